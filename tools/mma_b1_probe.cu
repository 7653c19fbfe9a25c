// Probe: throughput and fragment layout of mma.sync m16n8k256 b1 (and.popc) on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ void mma_b1(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
                 "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void tput(int iters, int* out, long long* cyc) {
    uint32_t a[8][4], b[2];
    int d[8][4];
    for (int c = 0; c < 8; ++c)
        for (int i = 0; i < 4; ++i) { a[c][i] = threadIdx.x * 77 + c * 13 + i; d[c][i] = 0; }
    b[0] = threadIdx.x; b[1] = ~threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) mma_b1(d[c], a[c], b);
    }
    long long t1 = clock64();
    int s = 0;
    for (int c = 0; c < 8; ++c) for (int i = 0; i < 4; ++i) s += d[c][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// layout probe: A [16 x 256] bits row-major (word w of row r = A[r*8 + w]), B [8 cols x 256] (word w of col n = B[n*8+w])
// guessed fragments: a0 = A[gid][tig], a1 = A[gid+8][tig], a2 = A[gid][4+tig], a3 = A[gid+8][4+tig]
//                    b0 = B[gid][tig], b1 = B[gid][4+tig];  d: c0,c1 = (gid, 2tig, 2tig+1), c2,c3 = (gid+8, ...)
__global__ void layout(const uint32_t* A, const uint32_t* B, int* D) {
    const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
    uint32_t a[4] = {A[gid * 8 + tig], A[(gid + 8) * 8 + tig], A[gid * 8 + 4 + tig], A[(gid + 8) * 8 + 4 + tig]};
    uint32_t b[2] = {B[gid * 8 + tig], B[gid * 8 + 4 + tig]};
    int d[4] = {0, 0, 0, 0};
    mma_b1(d, a, b);
    D[gid * 8 + 2 * tig] = d[0];
    D[gid * 8 + 2 * tig + 1] = d[1];
    D[(gid + 8) * 8 + 2 * tig] = d[2];
    D[(gid + 8) * 8 + 2 * tig + 1] = d[3];
}

int main() {
    int *out; long long* cyc;
    const int blocks = 148 * 4, threads = 128, iters = 4096;
    cudaMalloc(&out, blocks * threads * 4);
    cudaMalloc(&cyc, blocks * 8);
    tput<<<blocks, threads>>>(16, out, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tput<<<blocks, threads>>>(iters, out, cyc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(blocks); cudaMemcpy(c.data(), cyc, blocks * 8, cudaMemcpyDeviceToHost);
    double mmas = double(blocks) * (threads / 32) * iters * 8;
    printf("tput: %.3f ms, %.3e mma/s, %.2f mma/clk/SM (cycles/block %lld), bits/s(A) %.3e\n", ms, mmas / (ms * 1e-3),
           mmas / 148.0 / (c[0]), c[0], mmas * 4096 / (ms * 1e-3));
    // layout
    std::vector<uint32_t> A(16 * 8), B(8 * 8); std::vector<int> D(128), R(128);
    srand(1);
    for (auto& v : A) v = (uint32_t(rand()) << 16) ^ uint32_t(rand());
    for (auto& v : B) v = (uint32_t(rand()) << 16) ^ uint32_t(rand());
    uint32_t *dA, *dB; int* dD;
    cudaMalloc(&dA, 512); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
    cudaMemcpy(dA, A.data(), 512, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), 256, cudaMemcpyHostToDevice);
    layout<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(D.data(), dD, 512, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 16; ++r)
        for (int n = 0; n < 8; ++n) {
            int s = 0;
            for (int w = 0; w < 8; ++w) s += __builtin_popcount(A[r * 8 + w] & B[n * 8 + w]);
            if (s != D[r * 8 + n]) ++bad;
        }
    printf("layout mismatches: %d / 128 (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
    return 0;
}

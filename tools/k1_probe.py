"""K1 throughput vs the relative placement of base / fine buffers (DRAM channel conflicts?).
One Llama-2-70B layer set (7 matrices, bf16) compressed with one batched launch."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2402_10193_b200 as bd
from paper_2402_10193_b200 import capi

if len(sys.argv) > 1:  # a variant library (tools/k1var/build_variants.sh)
    capi.LIB_PATH = sys.argv[1]
dev = torch.device('cuda:0')
shapes = [(8192, 8192), (1024, 8192), (1024, 8192), (8192, 8192), (28672, 8192), (28672, 8192), (8192, 28672)]
params = sum(r * c for r, c in shapes)
algo = params * (4 + 1 / 8)


def timeit(pairs, reps=10):
    outs = [(torch.empty(bd.packed_size(*b.shape), dtype=torch.uint8, device=dev),
             torch.empty(1, dtype=torch.float32, device=dev)) for b, _ in pairs]
    for _ in range(3):
        bd.compress_batched(pairs, outs=outs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        bd.compress_batched(pairs, outs=outs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return algo / (ms / 1e3) / 1e9


big = torch.empty(2 * params + (64 << 20), dtype=torch.bfloat16, device=dev)
big.normal_()
for shift_kb in [0, 4096]:
    # all bases back to back, then all fines at +params + shift
    off = 0
    pairs = []
    fine_base = params + shift_kb * 512  # elements (2 B)
    for r, c in shapes:
        pairs.append((big[off:off + r * c].view(r, c), big[fine_base + off:fine_base + off + r * c].view(r, c)))
        off += r * c
    print(f"fine offset = params + {shift_kb} KB: {timeit(pairs):.0f} GB/s", flush=True)
# interleaved allocations like the bench
g = torch.Generator(device=dev).manual_seed(1)
for trial in range(2):
    pairs = []
    for r, c in shapes:
        b = torch.randn(r, c, device=dev, generator=g).to(torch.bfloat16)
        f = (b.float() + 1e-3).to(torch.bfloat16)
        pairs.append((b, f))
    print(f"separate allocations trial {trial}: {timeit(pairs):.0f} GB/s  "
          f"(fine-base offsets mod 2MB: {[(f.data_ptr() - b.data_ptr()) % (2 << 20) for b, f in pairs[:3]]})", flush=True)
    del pairs
    torch.cuda.empty_cache()

# the bench's f32 configs[0] shape: one 4096^2 pair, L2 swept between reps
b = torch.randn(4096, 4096, device=dev) * 0.02
f = b + 1e-3 * torch.randn_like(b)
outs = [(torch.empty(bd.packed_size(4096, 4096), dtype=torch.uint8, device=dev), torch.empty(1, device=dev))]
sweep = torch.ones(128 << 20, device=dev)
ts = []
for _ in range(20):
    sweep.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bd.compress_batched([(b, f)], outs=outs); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"f32 4096^2: median {4096 * 4096 * 8.125 / (ts[10] / 1e3) / 1e9:.0f} GB/s ({ts[10] * 1e3:.1f} us)")

import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2402_10193_b200 as bd
from test_gpu_kernels import _mt_reference, rel_l2
dev = torch.device("cuda:0")
rows, cols, B, T = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 1024, 1, 1))]
zero_w = len(sys.argv) > 5 and sys.argv[5] == "0"
torch.manual_seed(0)
W = (torch.randn(rows, cols, device=dev) * 0.02).to(torch.bfloat16)
if zero_w:
    W.zero_()
X = torch.randn(B, cols, device=dev).to(torch.bfloat16)
bits, al = [], []
for t in range(T):
    b, a = bd.compress_tensor(torch.zeros(rows, cols, device=dev), torch.randn(rows, cols, device=dev))
    bits.append(b); al.append(a.item())
rt = [b % T for b in range(B)]
Y = bd.multitenant_linear(W, bits, al, rt, X)
want = _mt_reference(W, bits, al, rt, X, rows, cols)
print("rel_l2", rel_l2(Y.cpu().numpy(), want.cpu().numpy()))
print(Y[0, :8].cpu().numpy()); print(want[0, :8].cpu().numpy())

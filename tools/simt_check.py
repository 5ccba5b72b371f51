import sys, torch
sys.path.insert(0, '.')
from paper_1806_03377_b200 import _native as nat
torch.manual_seed(0)
for (M, N, K, amn, bmn) in [(1024, 1024, 32, 1, 1), (1024, 1024, 64, 1, 1), (1024, 1024, 96, 1, 1), (32, 1024, 1024, 0, 1), (64, 1024, 1024, 0, 1), (64, 1024, 1024, 0, 0), (64, 256, 40, 1, 1)]:
    a = torch.randn((K, M) if amn else (M, K), device="cuda")
    b = torch.randn((K, N) if bmn else (N, K), device="cuda")
    A = (a.t() if amn else a).double(); Bm = (b.t() if bmn else b).double()
    ref = A @ Bm.t()
    out = torch.empty(M, N, device="cuda")
    nat.gemm(a, bool(amn), b, bool(bmn), M, N, K, kind=nat.EPI_STORE, out=out)
    m = torch.zeros(M, N, device="cuda"); ring = torch.empty(M, N, device="cuda")
    nat.gemm(a, bool(amn), b, bool(bmn), M, N, K, kind=nat.EPI_SGD, out=ring, master=m, lr=1.0)
    torch.cuda.synchronize()
    scale = (A.abs() @ Bm.abs().t())
    e1 = ((out.double() - ref).abs() / scale).max().item()
    e2 = ((-m.double() - ref).abs() / scale).max().item()
    print(M, N, K, amn, bmn, "store relerr %.2e" % e1, "sgd relerr %.2e" % e2)

import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
n = 130
X = torch.randn(n, n, n, dtype=torch.float64, device='cuda')
U = torch.randn(n, n, dtype=torch.float64, device='cuda')
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3
fl = 2 * n**4
for name, f in [("mode x (X@U)", lambda: X.reshape(-1, n) @ U),
                ("mode z (U@X)", lambda: U @ X.reshape(n, -1)),
                ("mode y batched (U@X[i])", lambda: torch.matmul(U, X))]:
    us = t(f); print(f"{name}: {us:.1f} us  {fl/us/1e6:.1f} TF")

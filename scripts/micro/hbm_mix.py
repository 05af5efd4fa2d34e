"""HBM bandwidth by read:write mix (diagnostic): write-only, 1:1 copy, 1:2 (one read, two writes)."""
import torch

def t(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

n = 1 << 30  # 4 GiB of fp32
a = torch.empty(n, device="cuda"); b = torch.empty(n, device="cuda"); c = torch.empty(n, device="cuda")
a.normal_()
ms = t(lambda: b.fill_(1.0)); print(f"write-only      {4*n/ms/1e6:8.0f} GB/s")
ms = t(lambda: b.copy_(a)); print(f"copy 1:1        {8*n/ms/1e6:8.0f} GB/s")
h = a.view(2, n // 2)
def split():
    torch.mul(a, 2.0, out=b); torch.mul(a, 3.0, out=c)
ms = t(split); print(f"2 x (1:1) back to back {16*n/ms/1e6:8.0f} GB/s")
bh = torch.empty(n, device="cuda", dtype=torch.float16); bl = torch.empty(n, device="cuda", dtype=torch.float16)
def hilo():
    bh.copy_(a)
ms = t(hilo); print(f"fp32 -> fp16 (1:0.5) {6*n/ms/1e6:8.0f} GB/s")
half = a[: n // 2]
ms = t(lambda: torch.cat([half, half], out=b)); print(f"cat 1:2 (read n/2, write n) {6*n/ms/1e6:8.0f} GB/s")

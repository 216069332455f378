"""HBM ceilings by read/write mix on one B200 (context for write-heavy kernels such as
k_tok_dispatch, which reads a row once and writes it k times): write-only (fill), copy (1:1),
and a 1-read : 8-write broadcast done by torch (index_copy-free: expand + copy)."""
import json
import torch

def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best

n = 1 << 31  # 4 GiB of bf16
y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
x = torch.empty(n // 8, dtype=torch.bfloat16, device="cuda").normal_()
src = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
out = {}
ms = t(lambda: y.fill_(1.0)); out["write_only_GBs"] = 2 * n / ms / 1e6
ms = t(lambda: y.copy_(src)); out["copy_GBs"] = 4 * n / ms / 1e6
yv = y.view(n // 8 // 2048, 8, 2048); xv = x.view(-1, 1, 2048)
ms = t(lambda: yv.copy_(xv.expand_as(yv))); out["bcast_1r8w_GBs"] = (2 * n + 2 * n // 8) / ms / 1e6
print(json.dumps(out))

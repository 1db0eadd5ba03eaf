"""HBM bandwidth probes for the traffic mixes of the row kernels (reference points, not the product)."""
import json, torch
torch.cuda.set_device(0)
n = 10 * 1024**3 // 2   # 10 GiB of bf16
x = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
y = torch.empty_like(x)
z = torch.empty(2 * n, dtype=torch.bfloat16, device="cuda")
def t(fn, nbytes, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return round(nbytes * it / a.elapsed_time(b) / 1e6, 1)
B = n * 2
res = {
  "copy_r1w1": t(lambda: y.copy_(x), 2 * B),
  "zero_w1": t(lambda: y.zero_(), B),
  "sum_r1": t(lambda: x.sum(dtype=torch.float32), B),
  "cat_r1w2": t(lambda: torch.cat([x, x], out=z), 3 * B),
}
print(json.dumps(res))

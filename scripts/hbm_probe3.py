"""The loss kernel's traffic mix (1 read : 2 writes) with better-fed probe kernels than hbm_probe2.py's
k_mix12 (one load in flight per thread): 4 loads in flight, and a row-structured copy / zero-fill mix shaped
like the math micro-batch. GB/s = bytes read + written / time (CUDA events)."""
import ctypes as C, json, subprocess, torch
so = "/tmp/hbm_kernels.so"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, "scripts/hbm_kernels.cu"])
L = C.CDLL(so)
torch.cuda.set_device(0)
nb = 8 * 1024**3
x = torch.empty(nb // 2, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x); z = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
def t(fn, nbytes, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return round(nbytes * it / a.elapsed_time(b) / 1e6, 1)
P = lambda t_: C.c_void_p(t_.data_ptr())
res = {}
res["copy_torch"] = t(lambda: y.copy_(x), 2 * nb)
for g in (1184, 2368):
    res[f"mix_r1w2_grid{g}"] = t(lambda: L.probe_mix12(P(x), P(y), P(z), C.c_size_t(nb), g, C.c_void_p(s)), 3 * nb)
    res[f"mix_r1w2_u4_grid{g}"] = t(lambda: L.probe_mix12_u4(P(x), P(y), P(z), C.c_size_t(nb), g, C.c_void_p(s)),
                                    3 * nb)
row = 151936 * 2
nrows = nb // row
rb = nrows * row
for g, th in ((148 * 2, 1024), (148 * 4, 512), (148 * 8, 256)):
    # mode 0: even rows read + write, odd rows write (3 row-bytes per 2 rows); 1: all rows copied; 2: all zero-filled
    for mode, by in ((0, rb * 3 // 2), (1, rb * 2), (2, rb)):
        res[f"rows_mode{mode}_grid{g}_t{th}"] = t(lambda: L.probe_mix_rows(P(x), P(y), C.c_size_t(rb), C.c_size_t(row),
                                                                          g, th, mode, C.c_void_p(s)), by)
print(json.dumps(res))

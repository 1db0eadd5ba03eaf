import ctypes as C, json, os, subprocess, torch
so = "/tmp/hbm_kernels.so"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, "scripts/hbm_kernels.cu"])
L = C.CDLL(so)
torch.cuda.set_device(0)
nb = 16 * 1024**3
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
for g in (148 * 4, 148 * 8, 148 * 16):
    res[f"stg_cs_w_grid{g}"] = t(lambda: L.probe_write_stg(P(y), C.c_size_t(nb), g, 0, C.c_void_p(s)), nb)
    res[f"stg_plain_w_grid{g}"] = t(lambda: L.probe_write_stg(P(y), C.c_size_t(nb), g, 1, C.c_void_p(s)), nb)
for ch in (4096, 16384, 65536):
    for g in (148, 296):
        res[f"bulk_w_chunk{ch}_grid{g}"] = t(lambda: L.probe_write_bulk(P(y), C.c_size_t(nb), g, ch, C.c_void_p(s)), nb)
o = torch.empty(148 * 16 * 512, dtype=torch.int32, device="cuda")
for g in (148 * 4, 148 * 8, 148 * 16):
    res[f"ldg_read_grid{g}"] = t(lambda: L.probe_read(P(x), C.c_size_t(nb), g, P(o), C.c_void_p(s)), nb)
for ch in (12288, 24576):
    for g in (148, 296):
        res[f"bulk_read_chunk{ch}_grid{g}"] = t(lambda: L.probe_read_bulk(P(x), C.c_size_t(nb), g, ch, P(o), C.c_void_p(s)), nb)
res["memset_w"] = t(lambda: L.probe_memset(P(y), C.c_size_t(nb), C.c_void_p(s)), nb)
res["mix_r1w2_grid1184"] = t(lambda: L.probe_mix12(P(x), P(y), P(z), C.c_size_t(nb), 1184, C.c_void_p(s)), 3 * nb)
res["mix_r1w2_grid2368"] = t(lambda: L.probe_mix12(P(x), P(y), P(z), C.c_size_t(nb), 2368, C.c_void_p(s)), 3 * nb)
print(json.dumps(res, indent=0))

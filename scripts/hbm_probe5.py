"""Zero-fill paths (round 2): cudaMemsetAsync (driver) vs an SM store kernel vs torch.zero_, alone and concurrently
with a copy kernel on another stream — does the driver's memset write faster than SM stores, and does it add to a
concurrent SM stream? GB/s = bytes written (+ read) / time, CUDA events, best of 3."""
import ctypes as C, json, os, sys, torch
sys.path.insert(0, os.getcwd())
import subprocess
so = "/tmp/hbm_kernels4.so"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, "scripts/hbm_kernels4.cu"])
L = C.CDLL(so)
cudart = C.CDLL(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so.12")) \
    if os.path.exists(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so.12")) else C.CDLL("libcudart.so")
torch.cuda.set_device(0)
nb = 4 * 1024**3
x = torch.empty(nb // 2, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x); z = torch.empty_like(x)
s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()
P = lambda t_: C.c_void_p(t_.data_ptr())
def memset(t, stream):
    return cudart.cudaMemsetAsync(P(t), 0, C.c_size_t(t.numel() * t.element_size()), C.c_void_p(stream.cuda_stream))
def t(fn, nbytes, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    best = 0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(it): fn()
        b.record(); torch.cuda.synchronize()
        best = max(best, nbytes * it / a.elapsed_time(b) / 1e6)
    return round(best, 1)
res = {}
res["memset_alone"] = t(lambda: memset(z, s0), nb)
res["zero_torch"] = t(lambda: z.zero_(), nb)
res["sm_write_coalesced"] = t(lambda: L.probe4_write_c(P(z), C.c_size_t(nb), 148, 1, C.c_void_p(s0.cuda_stream)), nb)
res["copy_sm"] = t(lambda: L.probe4_copy(P(x), P(y), C.c_size_t(nb), 148, 1, C.c_void_p(s0.cuda_stream)), 2 * nb)
def both():   # SM copy x -> y on s0 and a driver memset of z on s1, concurrently
    s1.wait_stream(s0)
    L.probe4_copy(P(x), P(y), C.c_size_t(nb), 148, 1, C.c_void_p(s0.cuda_stream))
    memset(z, s1)
    s0.wait_stream(s1)
res["copy_sm_plus_memset_concurrent"] = t(both, 3 * nb)
def both_sm():   # SM copy and SM zero-fill kernels on two streams
    s1.wait_stream(s0)
    L.probe4_copy(P(x), P(y), C.c_size_t(nb), 148, 1, C.c_void_p(s0.cuda_stream))
    L.probe4_write_c(P(z), C.c_size_t(nb), 148, 1, C.c_void_p(s1.cuda_stream))
    s0.wait_stream(s1)
res["copy_sm_plus_sm_zero_concurrent"] = t(both_sm, 3 * nb)
print(json.dumps(res))

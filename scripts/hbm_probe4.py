"""Store-path probes (round 2): pure write / copy / the loss kernel's row mix (the math micro-batch's trainable-row
pattern) with four store forms (0 st.global.cs.v4 = the row kernels' form, 1 plain st.global.v4, 2 256-bit
st.global.v8, 3 st.global.L1::no_allocate.v4), against torch copy_ and cudaMemsetAsync. GB/s = bytes read +
written / time (CUDA events, best of 3 x 5 launches). The *_sv0/1/3 write and rows forms store a thread's two
adjacent vectors with two instructions (each warp instruction half-fills its 32-byte sectors); *_coalesced_* store
lane-consecutive vectors (each warp instruction fills 512 contiguous bytes), the loss kernel's own pattern."""
import ctypes as C, json, os, subprocess, sys, torch
sys.path.insert(0, os.getcwd())
so = "/tmp/hbm_kernels4.so"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, "scripts/hbm_kernels4.cu"])
L = C.CDLL(so)
torch.cuda.set_device(0)
nb = 8 * 1024**3
x = torch.empty(nb // 2, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
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
P = lambda t_: C.c_void_p(t_.data_ptr())
res = {"copy_torch": t(lambda: y.copy_(x), 2 * nb), "zero_torch": t(lambda: y.zero_(), nb)}
# the math workload's trainable-row pattern (synth), rows of V = 151936 bf16
from synth import make_batch
tb = make_batch("math")
row = 151936 * 2
nrows = nb // row
import numpy as np
lm = np.zeros(int(tb.tok_offsets[-1]), dtype=np.uint8)
o = 0
for b in range(tb.num_traj):
    for sidx in range(int(tb.seg_offsets[b]), int(tb.seg_offsets[b + 1])):
        n = int(tb.seg_len[sidx])
        if int(tb.seg_source[sidx]) == 1:
            lm[o:o + n] = 1
        o += n
pat = torch.from_numpy(lm[:nrows].copy()).cuda()
frac = float(pat.float().mean())
rows_bytes = nrows * row * (1 + frac)
for g in (148, 296):
    for sv in range(4):
        res[f"write_sv{sv}_g{g}"] = t(lambda: L.probe4_write(P(y), C.c_size_t(nb), g, sv, C.c_void_p(s)), nb)
        res[f"copy_sv{sv}_g{g}"] = t(lambda: L.probe4_copy(P(x), P(y), C.c_size_t(nb), g, sv, C.c_void_p(s)), 2 * nb)
        res[f"rows_sv{sv}_g{g}"] = t(lambda: L.probe4_rows(P(x), P(y), C.c_size_t(nrows), C.c_size_t(row), P(pat), g,
                                                           sv, C.c_void_p(s)), rows_bytes)
for g in (148, 296):
    for sv in (0, 1):
        res[f"write_coalesced_sv{sv}_g{g}"] = t(lambda: L.probe4_write_c(P(y), C.c_size_t(nb), g, sv, C.c_void_p(s)), nb)
        res[f"rows_coalesced_sv{sv}_g{g}"] = t(lambda: L.probe4_rows_c(P(x), P(y), C.c_size_t(nrows), C.c_size_t(row),
                                                                       P(pat), g, sv, C.c_void_p(s)), rows_bytes)
res["rows_trainable_frac"] = round(frac, 4)
print(json.dumps(res))

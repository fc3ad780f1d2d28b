# c1 SpMM event time per library variant (AUTOSAGE_DEV_LIB), cold L2 per call
for lib in paper_2511_17594_b200/libautosage_b200_lv_*.so; do
AUTOSAGE_DEV_LIB=$PWD/$lib python - "$lib" <<'PY'
import os, sys, ctypes as C, torch
sys.path.insert(0, os.getcwd())
import bench, paper_2511_17594_b200 as asb
from paper_2511_17594_b200 import _capi
m, f = bench.make_graph("c1", 1)
b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).cuda()
g = asb.Graph.from_csr(m)
c = torch.empty((m.n_rows, f), device="cuda")
s = asb.torch_stream_handle()
flush = torch.empty(64 << 20, device="cuda")
out = []
for vs in ("spmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256", "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"):
    v = asb.variant_from_string(vs).to_c()
    run = lambda: asb._check(_capi.lib.as_spmm(C.byref(v), g.handle, C.c_void_p(b.data_ptr()), m.n_cols, f,
                                               C.c_void_p(c.data_ptr()), C.c_void_p(s), None))
    for _ in range(5): run()
    ts = []
    for _ in range(50):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); out.append(f"{vs.split(':')[1]} {ts[len(ts)//2]:.4f}")
print(os.path.basename(sys.argv[1]), "  ".join(out))
PY
done

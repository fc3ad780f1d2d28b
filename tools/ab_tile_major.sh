# SpMM tile-major item order A/B at F = 128 / 256 (Reddit-shape), fixed variants, cold L2
for tm in 1 0 1 0; do
AUTOSAGE_DEV_TILE_MAJOR=$tm python - <<'PY'
import os, sys, ctypes as C, torch
sys.path.insert(0, os.getcwd())
import bench, paper_2511_17594_b200 as asb
from paper_2511_17594_b200 import _capi
m, _ = bench.make_graph("reddit", 1)
g = asb.Graph.from_csr(m)
s = asb.torch_stream_handle()
flush = torch.empty(64 << 20, device="cuda")
out = []
for f in (128, 256):
    b = torch.from_numpy(asb.fill_uniform(m.n_cols * f, 1 + f, (m.n_cols, f))).cuda()
    c = torch.empty((m.n_rows, f), device="cuda")
    for vs in (f"spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256", f"spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256", f"spmm:hubsplit:ft={f}:rpc=1:vec=1:hubt=256"):
        v = asb.variant_from_string(vs).to_c()
        run = lambda: asb._check(_capi.lib.as_spmm(C.byref(v), g.handle, C.c_void_p(b.data_ptr()), m.n_cols, f,
                                                   C.c_void_p(c.data_ptr()), C.c_void_p(s), None))
        run()
        ts = []
        for _ in range(7):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        out.append(f"F={f} ft={vs.split('ft=')[1].split(':')[0]} {sorted(ts)[3]:.3f}")
    del b, c
print(f"tile_major={os.environ['AUTOSAGE_DEV_TILE_MAJOR']}:", "  ".join(out), flush=True)
PY
done

# c1 SpMM latency vs the long-row threshold / fork knobs (one process per setting: knobs are read once)
for lr in 256 128 64 32; do
  for conc in 1 0; do
    AUTOSAGE_DEV_LONG_ROW=$lr AUTOSAGE_DEV_SPMM_CONCURRENT=$conc python - <<'PY'
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
for vs in ("spmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256", "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256",
           "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=64"):
    v = asb.variant_from_string(vs).to_c()
    run = lambda: asb._check(_capi.lib.as_spmm(C.byref(v), g.handle, C.c_void_p(b.data_ptr()), m.n_cols, f,
                                               C.c_void_p(c.data_ptr()), C.c_void_p(s), None))
    for _ in range(5): run()
    ts = []
    for _ in range(50):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); out.append(f"{vs.split(':')[1]}/hubt={vs.split('=')[-1]} {ts[len(ts)//2]:.4f}")
print(f"long_row={os.environ['AUTOSAGE_DEV_LONG_ROW']} conc={os.environ['AUTOSAGE_DEV_SPMM_CONCURRENT']}:", "  ".join(out))
PY
  done
done

"""Developer timing of wn_build_faces (+ one query) on C5 (not the bench contract).
WN_LIB_OVERRIDE selects a library variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25159_b200 as wn  # noqa: E402
from wn_workloads import configs as G  # noqa: E402

wl = G.gen_c5()
dev = torch.device("cuda", 0)
T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
geo = [T(wl["ctrl_uv"], torch.float64), T(wl["ctrl_w"], torch.float64), T(wl["seg_degree"], torch.int32),
       T(wl["loop_seg_off"], torch.int32), T(wl["face_loop_off"], torch.int32), T(wl["face_periodic"], torch.uint8),
       T(wl["face_domain"], torch.float64)]
fid, uv = T(wl["face_id"], torch.int32), T(wl["uv"], torch.float64)
w = torch.empty(len(fid), dtype=torch.float64, device=dev)
f = torch.empty(len(fid), dtype=torch.uint8, device=dev)
for _ in range(3):
    wn.Faces.build(*geo).close()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
a.record()
for _ in range(K):
    wn.Faces.build(*geo).close()
b.record()
torch.cuda.synchronize()
tb = a.elapsed_time(b) / K
fc = wn.Faces.build(*geo)
fc.query(fid, uv, out=(w, f))
torch.cuda.synchronize()
a.record()
for _ in range(K):
    fc.query(fid, uv, out=(w, f))
b.record()
torch.cuda.synchronize()
tq = a.elapsed_time(b) / K
fc.set_counters(True)
fc.query(fid, uv, out=(w, f))
c = fc.counters()
fc.close()
print("%s build %.3f ms  query %.3f ms  inside %d  warp_records %d span %d pairs %d hard %d nodes %d" % (
    os.path.basename(os.environ.get("WN_LIB_OVERRIDE", "libwn.so")), tb, tq, int(f.sum().item()), c["warp_records"],
    c["span_tests"], c["pairs_tested"], c["hard_pairs"], c["nodes"]))

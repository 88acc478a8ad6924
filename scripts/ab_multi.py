#!/usr/bin/env python
"""A/B timing of libwn variants in ONE process (the C5 batch generated once):
    python scripts/ab_multi.py path/to/libA.so path/to/libB.so ...
Per variant: build (wn_build_faces) and query (wn_query) CUDA-event times over
K repetitions, interleaved rounds, plus the work counters and the K3 split."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25159_b200 as wn  # noqa: E402
from wn_workloads import configs as G  # noqa: E402

libs = sys.argv[1:]
cfg = os.environ.get("AB_CFG", "C5")
wl = {"C5": lambda: G.gen_c5(), "C2": lambda: G.gen_c2(), "C3": lambda: G.gen_c3()}[cfg]()
dev = torch.device("cuda", 0)
T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
geo = [T(wl["ctrl_uv"], torch.float64), T(wl["ctrl_w"], torch.float64), T(wl["seg_degree"], torch.int32),
       T(wl["loop_seg_off"], torch.int32), T(wl["face_loop_off"], torch.int32), T(wl["face_periodic"], torch.uint8),
       T(wl["face_domain"], torch.float64)]
fid, uv = T(wl["face_id"], torch.int32), T(wl["uv"], torch.float64)
n = len(fid)
w = torch.empty(n, dtype=torch.float64, device=dev)
f = torch.empty(n, dtype=torch.uint8, device=dev)
ref = None


def use(path):
    wn._lib = None
    wn._LIBPATH = path
    wn.load()


def run(path, K=10):
    use(path)
    for _ in range(3):
        wn.Faces.build(*geo).close()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        wn.Faces.build(*geo).close()
    b.record()
    torch.cuda.synchronize()
    tb = a.elapsed_time(b) / K
    fc = wn.Faces.build(*geo)
    fc.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    fc.set_timing(True)
    a.record()
    for _ in range(K):
        fc.query(fid, uv, out=(w, f))
    b.record()
    torch.cuda.synchronize()
    tq = a.elapsed_time(b) / K
    k3, p1, kn = fc.timing()
    fc.set_timing(False)
    a.record()
    for _ in range(K):
        g = wn.Faces.build(*geo)
        g.query(fid, uv, out=(w, f))
        g.close()
    b.record()
    torch.cuda.synchronize()
    ts = a.elapsed_time(b) / K
    fc.set_counters(True)
    fc.query(fid, uv, out=(w, f))
    c = fc.counters()
    fc.close()
    return tb, tq, ts, k3 / max(kn, 1), p1 / max(kn, 1), c, f.clone(), w.clone()


res = {p: [] for p in libs}
for rnd in range(3):
    for p in libs:
        res[p].append(run(p))
for p in libs:
    r = res[p]
    tb = min(x[0] for x in r); tq = min(x[1] for x in r); ts = min(x[2] for x in r)
    k3 = min(x[3] for x in r); p1 = min(x[4] for x in r)
    c = r[-1][5]
    fl, wv = r[-1][6], r[-1][7]
    if ref is None:
        ref = (fl, wv)
        same = "ref"
    else:
        same = "flags %s, winding max|d| %.3g" % ("identical" if torch.equal(fl, ref[0]) else "DIFFER (%d)" % int((fl != ref[0]).sum()),
                                                  float(torch.nan_to_num(wv - ref[1], nan=0.0).abs().max()))
    print("%-34s build %.3f  query %.3f  step %.3f  k3 %.3f  p1 %.3f  hard %.3f | warp_it %d lane_tests %d hard %d nodes %d | %s" % (
        os.path.basename(p), tb, tq, ts, k3, p1, k3 - p1, c["warp_records"], c["pairs_tested"] + c["span_tests"],
        c["hard_pairs"], c["nodes"], same), flush=True)

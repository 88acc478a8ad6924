#!/usr/bin/env python
"""A/B of runtime switches (environment variables read per call) in ONE process:
    python scripts/ab_env.py "" "WN_HARD1=0" "WN_HARD1=0 WN_FINISH_Q=0"
Per setting: query / step CUDA-event times, the K3 split, and the results
compared with the first setting's."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25159_b200 as wn  # noqa: E402
from wn_workloads import configs as G  # noqa: E402

settings = sys.argv[1:] or [""]
cfg = os.environ.get("AB_CFG", "C5")
wl = {"C5": G.gen_c5, "C2": G.gen_c2, "C3": G.gen_c3, "C4": G.gen_c4, "C1": G.gen_c1}[cfg]()
dev = torch.device("cuda", 0)
T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
geo = [T(wl["ctrl_uv"], torch.float64), T(wl["ctrl_w"], torch.float64), T(wl["seg_degree"], torch.int32),
       T(wl["loop_seg_off"], torch.int32), T(wl["face_loop_off"], torch.int32), T(wl["face_periodic"], torch.uint8),
       T(wl["face_domain"], torch.float64)]
fid, uv = T(wl["face_id"], torch.int32), T(wl["uv"], torch.float64)
n = len(fid)
w = torch.empty(n, dtype=torch.float64, device=dev)
f = torch.empty(n, dtype=torch.uint8, device=dev)


def run(setting, K=10):
    keys = []
    for kv in setting.split():
        k, v = kv.split("=")
        os.environ[k] = v
        keys.append(k)
    fc = wn.Faces.build(*geo)
    fc.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    fc.set_timing(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fc.query(fid, uv, out=(w, f))
    b.record()
    torch.cuda.synchronize()
    tq = a.elapsed_time(b) / K
    k3, p1, kn = fc.timing()
    fc.set_timing(False)
    fc.set_counters(True)
    fc.query(fid, uv, out=(w, f))
    c = fc.counters()
    fc.set_counters(False)
    fc.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    fc.close()
    for k in keys:
        del os.environ[k]
    return tq, k3 / max(kn, 1), p1 / max(kn, 1), c, f.clone(), w.clone()


res = {s: [] for s in settings}
for rnd in range(3):
    for s in settings:
        res[s].append(run(s))
ref = None
for s in settings:
    r = res[s]
    tq = min(x[0] for x in r); k3 = min(x[1] for x in r); p1 = min(x[2] for x in r)
    c, fl, wv = r[-1][3], r[-1][4], r[-1][5]
    if ref is None:
        ref = (fl, wv, c)
        same = "ref"
    else:
        same = "flags %s, winding max|d| %.3g, counters %s" % (
            "identical" if torch.equal(fl, ref[0]) else "DIFFER (%d)" % int((fl != ref[0]).sum()),
            float(torch.nan_to_num(wv - ref[1], nan=0.0).abs().max()), "identical" if c == ref[2] else "DIFFER")
    print("%-28s query %.3f  k3 %.3f  p1 %.3f  rest %.3f | hard %d nodes %d evals %d leaves %d | %s" % (
        s or "(default)", tq, k3, p1, k3 - p1, c["hard_pairs"], c["nodes"], c["evals"], c["leaves"], same), flush=True)

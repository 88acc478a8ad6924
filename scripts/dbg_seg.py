import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2510_25159_b200 as wn
from wn_workloads import configs as G
from tests import helpers as H
wl = G.gen_c2(n_queries=5000)
pts = np.array([[0.7051672636988958, 0.8489820320481127], [0.28714554050794244, 0.8050997279035224], [0.7030933974160354, 0.39744534071761367]])
loops = H.loops_of(wl)
segs = [s for l in loops for s in l]
faces = [([[s]], 0, (0, 1, 0, 1)) for s in segs]
fid = np.repeat(np.arange(len(segs)), len(pts)); q = np.tile(pts, (len(segs), 1))
wl1 = H.make_wl(faces, q, fid)
for am in (0, 1):
    f = wn.Faces.from_workload(wl1, angle_mode=am)
    f.set_counters(True)
    r = f.query(wl1["face_id"], wl1["uv"]); torch.cuda.synchronize()
    w = r.winding.cpu().numpy()
    print("angle", am, f.counters())
    for i, (P, wt) in enumerate(segs):
        for k, p in enumerate(pts):
            ref = oracle.segment_winding(P, wt, p)[0]
            g = w[i * len(pts) + k]
            if not abs(g - ref) < 1e-9:
                print("seg", i, "pt", k, "gpu", g, "ref", ref, "deg", len(P) - 1, "P", P.tolist(), "w", wt.tolist())
    f.close()
out = wn.segment_prep(wl["ctrl_uv"], wl["ctrl_w"], wl["seg_degree"]).cpu().numpy()
np.save("gpurun_out/c2_prep.npy", out)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2510_25159_b200 as wn
from wn_workloads import configs as G
for name, wl in [("C1", G.gen_c1(n_queries=5000)), ("C3", G.gen_c3(n_queries=5000)), ("C2", G.gen_c2(n_queries=5000))]:
    ref = oracle.query(wl); cm = ref["comparable"]
    for cap in ["1", "64", "1000000"]:
        os.environ["WN_HQ_CAP"] = cap
        for am in (0, 1):
            f = wn.Faces.from_workload(wl, angle_mode=am)
            r = f.query(wl["face_id"], wl["uv"]); torch.cuda.synchronize()
            w = r.winding.cpu().numpy(); fl = r.flag.cpu().numpy()
            bad = np.nonzero(cm & (fl != ref["flag"]))[0]
            err = np.nanmax(np.abs(w[cm] - ref["w"][cm]))
            print(name, "cap", cap, "angle", am, "mismatch", len(bad), "maxerr", err, flush=True)
            if len(bad): print("   ", wl["uv"][bad[:3]].tolist(), w[bad[:3]], ref["w"][bad[:3]])
            f.close()

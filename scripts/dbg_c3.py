import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2510_25159_b200 as wn
from wn_workloads import configs as G
wl = G.gen_c3(n_queries=20000)
ref = oracle.query(wl)
cm = ref["comparable"]
for dbg in ["0", "1", "2", "3"]:
    os.environ["WN_DBG"] = dbg
    for am in (0, 1):
        f = wn.Faces.from_workload(wl, angle_mode=am)
        f.set_counters(True)
        r = f.query(wl["face_id"], wl["uv"]); torch.cuda.synchronize()
        w = r.winding.cpu().numpy(); fl = r.flag.cpu().numpy()
        bad = np.nonzero(cm & (fl != ref["flag"]))[0]
        print("dbg", dbg, "angle", am, "mismatch", len(bad), "maxerr", np.nanmax(np.abs(w[cm]-ref["w"][cm])), f.counters())
        if len(bad): print("  e.g.", wl["uv"][bad[:3]], w[bad[:3]], ref["w"][bad[:3]])
        f.close()

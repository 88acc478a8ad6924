"""Experiment: K3 time vs sub-tiles per CTA unit (WN_SUBTILES) on C5."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_25159_b200 as wn
from wn_workloads import configs as G

wl = G.gen_c5()
faces = wn.Faces.from_workload(wl)
fid = torch.from_numpy(wl["face_id"]).cuda(); uv = torch.from_numpy(wl["uv"]).cuda()
n = fid.numel()
w = torch.empty(n, dtype=torch.float64, device="cuda"); f = torch.empty(n, dtype=torch.uint8, device="cuda")
ref = None
for s in sys.argv[1:] or ["1", "2", "4", "8", "16"]:
    os.environ["WN_SUBTILES"] = s
    for _ in range(2): faces.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    faces.set_timing(True)
    for _ in range(5): faces.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    k3, p1, nq = faces.timing(); faces.set_timing(False)
    wc = w.cpu().numpy(); fc = f.cpu().numpy()
    if ref is None: ref = (wc.copy(), fc.copy())
    same = np.array_equal(fc, ref[1]) and np.allclose(np.nan_to_num(wc, nan=7.0), np.nan_to_num(ref[0], nan=7.0), atol=1e-9, rtol=0)
    print(f"sub={s:3s} k3={k3/5:.3f} ms phase1={p1/5:.3f} ms same={same}", flush=True)

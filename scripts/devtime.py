"""Developer timing of wn_query on the configs (not the bench contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_25159_b200 as wn
from wn_workloads import configs as G

def run(name, wl, reps=5, **kw):
    t0 = time.time()
    faces = wn.Faces.from_workload(wl, **kw)
    torch.cuda.synchronize(); tb = time.time() - t0
    fid = torch.from_numpy(wl["face_id"]).cuda(); uv = torch.from_numpy(wl["uv"]).cuda()
    n = fid.numel()
    w = torch.empty(n, dtype=torch.float64, device="cuda"); f = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2): faces.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); faces.query(fid, uv, out=(w, f)); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    faces.set_counters(True); faces.query(fid, uv, out=(w, f)); c = faces.counters(); faces.set_counters(False)
    t = min(ts)
    pairs = G.n_input_pairs(wl)
    print(f"{name:10s} n={n:>9d} build={tb*1e3:8.1f} ms query={t:8.3f} ms  {n/t/1e6:8.2f} Gq/s... q/s={n/(t/1e3):.3e} pairs/s={pairs/(t/1e3):.3e} info={faces.info()} counters={c} flags={np.bincount(f.cpu().numpy(), minlength=4)}", flush=True)
    faces.close()

cfgs = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
for c in cfgs:
    t = time.time(); wl = G.CONFIGS[c](); print(c, "gen", time.time() - t, flush=True)
    run(c, wl)
    if c == "C4":
        run("C4-fp32", G.to_fp32_inputs(wl), precision=1)
    if c in ("C2", "C5"):
        run(c + "-angle", wl, angle_mode=1); run(c + "-flat", wl, hierarchy=False)

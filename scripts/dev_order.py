"""Experiment: effect of query order within a face on K3 (C5 grid queries)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_25159_b200 as wn
from wn_workloads import configs as G

wl = G.gen_c5()
faces = wn.Faces.from_workload(wl)
fid0 = wl["face_id"]; uv0 = wl["uv"]
n = fid0.size
g = 64
r = np.arange(g)[:, None].repeat(g, 1).ravel(); c = np.arange(g)[None, :].repeat(g, 0).ravel()
def morton(x, y):
    k = np.zeros_like(x)
    for b in range(6):
        k |= ((x >> b) & 1) << (2 * b); k |= ((y >> b) & 1) << (2 * b + 1)
    return k
orders = {
    "rowmajor": np.arange(g * g),
    "tile8x4": np.lexsort((c % 8, r % 4, c // 8, r // 4)),
    "morton": np.argsort(morton(c, r), kind="stable"),
    "random": np.random.default_rng(0).permutation(g * g),
}
nf = n // (g * g)
base = (np.arange(nf) * g * g)[:, None]
for name, o in orders.items():
    perm = (base + o[None, :]).ravel()
    fid = torch.from_numpy(fid0[perm]).cuda(); uv = torch.from_numpy(np.ascontiguousarray(uv0[perm])).cuda()
    w = torch.empty(n, dtype=torch.float64, device="cuda"); f = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2): faces.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    faces.set_timing(True)
    for _ in range(5): faces.query(fid, uv, out=(w, f))
    torch.cuda.synchronize()
    k3, p1, nq = faces.timing(); faces.set_timing(False)
    faces.set_counters(True); faces.query(fid, uv, out=(w, f)); cn = faces.counters(); faces.set_counters(False)
    print(f"{name:9s} k3={k3/5:.3f} ms phase1={p1/5:.3f} ms counters={cn}", flush=True)

#!/usr/bin/env python
"""Small end-to-end program for compute-sanitizer (memcheck / racecheck /
synccheck): every libwn kernel family at reduced sizes -- K1/K2 build incl. the
device planner and the bi-periodic pairing probes, K4 bucketing (sorted and
unsorted batches), k_phase1 with TMA staging (single- and multi-chunk faces),
the per-warp hard-pair buffers and the global queue (also forced to overflow:
k_overflow), k_hard, k_finish, the implicit-grid path, the NURBS ingest, fp32
records.  Checks the results against the oracle so a run that "passes" the
sanitizer also computed the right thing.

    compute-sanitizer --tool memcheck python scripts/sanitize_target.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2510_25159_b200 as wn  # noqa: E402
from tests import helpers as H  # noqa: E402
from wn_workloads import configs as G  # noqa: E402


def check(wl, w, fl, fp32=False):
    delta, tol = (1e-5, 1e-4) if fp32 else (1e-9, 1e-9)
    r = oracle.query(wl, delta=delta, tol=tol)
    cm = r["comparable"]
    assert np.array_equal(fl[cm], r["flag"][cm]), "flag mismatch"
    assert np.max(np.abs(w[cm] - r["w"][cm])) <= tol
    return int(cm.sum())


def run(wl, **kw):
    faces = wn.Faces.from_workload(wl, **kw)
    r = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    out = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    return out


def main():
    small = os.environ.get("WN_SAN_SMALL", "0") == "1"
    sc = 4 if small else 1
    cases = [
        ("C1", G.gen_c1(n_queries=4096 // sc), {}),
        ("C2", G.gen_c2(n_queries=20_000 // sc), {}),
        ("C2-angle", G.gen_c2(n_queries=8_000 // sc), dict(angle_mode=1)),
        ("C3", G.gen_c3(n_queries=6_000 // sc), {}),
        ("C3-generic", G.gen_c3(n_queries=6_000 // sc, exact=False, store_jitter=2), {}),
        ("C3pq", G.gen_c3pq(p=3, q=-2, n_queries=4_000 // sc, exact=False, store_jitter=2), dict(hierarchy=False)),
        ("C4-fp32", G.to_fp32_inputs(G.gen_c4(n_faces=60, n_deleted=6)), dict(precision=1)),
        ("C5", G.gen_c5(n_faces=60, grid=16, exact=False, store_jitter=1), {}),
    ]
    for name, wl, kw in cases:
        w, fl = run(wl, **kw)
        n = check(wl, w, fl, fp32=kw.get("precision", 0) == 1)
        print("%-10s ok (%d comparable)" % (name, n), flush=True)
    # unsorted batch (K4 scatter + spatial regrouping)
    wl = G.gen_c4(n_faces=30, q_per_face=300, n_deleted=3)
    perm = np.random.default_rng(2).permutation(len(wl["face_id"]))
    wl2 = dict(wl)
    wl2["face_id"], wl2["uv"] = wl["face_id"][perm], wl["uv"][perm]
    w, fl = run(wl2)
    print("unsorted   ok (%d comparable)" % check(wl2, w, fl), flush=True)
    # multi-chunk face (record program > 32 KB of shared memory)
    rng = np.random.default_rng(12)
    from wn_workloads.configs import _star_segments, _star_vertices
    outer = _star_segments(rng, _star_vertices(rng, (0.5, 0.5), 0.42, 0.02, 3000, False),
                           rng.integers(1, 6, 3000), 0.05, True)
    q = rng.uniform(0.05, 0.95, size=(2_000 // sc, 2))
    wl = H.make_wl([([outer], 0, (0, 1, 0, 1))], q)
    w, fl = run(wl)
    print("multichunk ok (%d comparable)" % check(wl, w, fl), flush=True)
    # forced hard-pair queue overflow: k_overflow
    os.environ["WN_HQ_CAP"] = "64"
    wl = G.gen_c2(n_queries=3_000 // sc)
    w, fl = run(wl)
    print("overflow   ok (%d comparable)" % check(wl, w, fl), flush=True)
    del os.environ["WN_HQ_CAP"]
    # implicit grids
    wl = G.gen_c5(n_faces=40, grid=16)
    gb = wl["meta"]["grid_box"]
    faces = wn.Faces.from_workload(wl)
    r = faces.query_grid(np.arange(len(gb)), gb, 16, 16)
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    print("grid       ok (%d comparable)" % check(wl, w, fl), flush=True)
    # NURBS ingest
    wl = G.gen_nurbs(n_faces=20, q_per_face=64)
    faces = wn.Faces.from_nurbs_workload(wl)
    r = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    print("nurbs      ok (%d comparable)" % check(oracle.nurbs_to_bezier_workload(wl), w, fl), flush=True)
    print("SANITIZE TARGET DONE")


if __name__ == "__main__":
    main()

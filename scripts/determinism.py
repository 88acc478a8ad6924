#!/usr/bin/env python
"""Determinism across launch configurations (a racecheck substitute: the
pool's compute-sanitizer is closed).  Every query's result is a permutation-
and schedule-invariant function of the inputs in crossing mode (integer sums),
so the same batch run (a) twice, (b) with 1 / 4 / 16 sub-tiles per unit,
(c) with and without the Morton regrouping, (d) from a shuffled batch must give
bit-identical flags and windings.  A shared-memory race (record staging,
hard-pair buffers, regrouping histogram) or a read of unwritten memory (with
WN_ALLOC_POISON=1) shows up as a difference."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25159_b200 as wn  # noqa: E402
from wn_workloads import configs as G  # noqa: E402


def run(wl, env, perm=None):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        faces = wn.Faces.from_workload(wl)
        fid, uv = wl["face_id"], wl["uv"]
        if perm is not None:
            fid, uv = fid[perm], uv[perm]
        r = faces.query(fid, uv)
        torch.cuda.synchronize()
        w, f = r.winding.cpu().numpy(), r.flag.cpu().numpy()
        faces.close()
        if perm is not None:
            inv = np.empty_like(perm)
            inv[perm] = np.arange(len(perm))
            w, f = w[inv], f[inv]
        return w, f
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def same(a, b, tol=0.0):
    if not np.array_equal(a[1], b[1]):
        return False
    wa, wb = np.nan_to_num(a[0], nan=7.0), np.nan_to_num(b[0], nan=7.0)
    return np.array_equal(wa, wb) if tol == 0.0 else bool(np.max(np.abs(wa - wb)) <= tol)


def main():
    cases = {"C2": G.gen_c2(n_queries=200_000), "C3-generic": G.gen_c3(n_queries=100_000, exact=False, store_jitter=2),
             "C5": G.gen_c5(n_faces=2000, grid=32, exact=False, store_jitter=1),
             "C4": G.gen_c4(n_faces=400, n_deleted=40)}
    bad = 0
    for name, wl in cases.items():
        ref = run(wl, {})
        variants = [("repeat", {}, None)] + [("subtiles=%d" % k, {"WN_SUBTILES": str(k)}, None) for k in (1, 4, 16)]
        variants += [("no-regroup", {"WN_NO_SPATIAL": "1"}, None),
                     ("shuffled", {}, np.random.default_rng(5).permutation(len(wl["face_id"]))),
                     ("queue-overflow", {"WN_HQ_CAP": "4096"}, None)]
        for vname, env, perm in variants:
            # k_overflow recomputes a query serially: its integer and fractional
            # terms are summed in another order than phase 1 + k_hard's atomic
            # adds, so windings may differ in the last bits (flags may not)
            tol = 1e-12 if vname == "queue-overflow" else 0.0
            ok = same(ref, run(wl, env, perm), tol)
            bad += not ok
            print("%-11s %-15s %s" % (name, vname, "identical" if ok else "DIFFERENT"), flush=True)
    print("DETERMINISM %s" % ("OK" if bad == 0 else "FAILED (%d)" % bad))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

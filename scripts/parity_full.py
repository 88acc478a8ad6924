#!/usr/bin/env python
"""Full-size GPU <-> oracle parity report (SURVEY 8(c) "Comparison rules"):
every query of every BASELINE config (no subsampling) through the C ABI in the
bench launch configuration, against the full CPU oracle on the host cores.

    python scripts/parity_full.py [--out PARITY_r02.json] [--configs C1,C2,...]

Per config it records: n, the oracle's comparable / excluded counts, flag
mismatches on comparable queries (must be 0), max and p99.99 |d omega| there,
the GPU on-boundary / invalid counts on comparable queries (must be 0), the
GPU on-boundary count overall and the oracle's wall time.  fp64 configs:
delta = tol = 1e-9; C4-fp32: oracle on the fp32-rounded inputs, delta = 1e-5,
tol = 1e-4 (reading R19).  "-generic" variants: periodic data as plain fp64
(T = 2 pi unquantised, random storage translates; wn_workloads exact=False).
Exit status 1 if any config fails the contract.
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def configs():
    from wn_workloads import configs as G
    return {
        "C1": (lambda: G.gen_c1(), 0),
        "C2": (lambda: G.gen_c2(), 0),
        "C3": (lambda: G.gen_c3(), 0),
        "C3-generic": (lambda: G.gen_c3(exact=False, store_jitter=2), 0),
        "C3pq(3,-2)-generic": (lambda: G.gen_c3pq(p=3, q=-2, n_queries=200_000, exact=False, store_jitter=2,
                                                  beta_shift=(2, -1)), 0),
        "C4": (lambda: G.gen_c4(), 0),
        "C4-fp32": (lambda: G.to_fp32_inputs(G.gen_c4()), 1),
        "C5": (lambda: G.gen_c5(), 0),
        "C5-generic": (lambda: G.gen_c5(exact=False, store_jitter=2), 0),
    }


def run_one(name, gen, precision):
    import torch
    import oracle
    import paper_2510_25159_b200 as wn
    t = time.time()
    wl = gen()
    t_gen = time.time() - t
    faces = wn.Faces.from_workload(wl, precision=precision)
    r = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    info = faces.info()
    faces.close()
    del r
    delta, tol = (1e-5, 1e-4) if precision else (1e-9, 1e-9)
    t = time.time()
    ref = oracle.query(wl, delta=delta, tol=tol)
    t_or = time.time() - t
    cm = ref["comparable"]
    n = len(w)
    err = np.abs(w[cm] - ref["w"][cm])
    err = err[np.isfinite(err)] if err.size else err
    mism = int(np.count_nonzero(fl[cm] != ref["flag"][cm]))
    onb_c = int(np.count_nonzero(fl[cm] == 2))
    inv_c = int(np.count_nonzero(fl[cm] == 3))
    nan_c = int(np.count_nonzero(~np.isfinite(w[cm])))
    res = {
        "n": n, "comparable": int(cm.sum()), "excluded": int(n - cm.sum()),
        "excluded_frac": float(1 - cm.mean()),
        "flag_mismatch": mism, "gpu_on_boundary_on_comparable": onb_c, "gpu_invalid_on_comparable": inv_c,
        "gpu_nan_on_comparable": nan_c,
        "max_abs_dw": float(err.max()) if err.size else 0.0,
        "p9999_abs_dw": float(np.quantile(err, 0.9999)) if err.size else 0.0,
        "tol": tol, "delta": delta, "precision": "fp32" if precision else "fp64",
        "gpu_on_boundary_total": int(np.count_nonzero(fl == 2)),
        "inside_frac": float(np.mean(fl == 1)),
        "records": info["n_records"], "seg_records": info["n_seg_records"],
        "oracle_s": t_or, "generate_s": t_gen,
    }
    res["pass"] = bool(mism == 0 and onb_c == 0 and inv_c == 0 and nan_c == 0 and res["max_abs_dw"] <= tol)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "PARITY_r02.json"))
    ap.add_argument("--configs", default=None)
    args = ap.parse_args()
    import torch
    allc = configs()
    names = list(allc) if not args.configs else args.configs.split(",")
    out = {"what": "full-size GPU vs oracle parity, every query (SURVEY 8(c) comparison rules)",
           "gpu": torch.cuda.get_device_name(0), "host": platform.processor() or platform.machine(),
           "cores": os.cpu_count(), "configs": {}}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    out["host"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ok = True
    for nm in names:
        gen, prec = allc[nm]
        res = run_one(nm, gen, prec)
        out["configs"][nm] = res
        ok &= res["pass"]
        print(nm, json.dumps(res), flush=True)
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)
    out["all_pass"] = bool(ok)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())

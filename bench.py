#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for libwn (arXiv 2510.25159 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl wn|reference]

Metric (BASELINE.json): winding-number queries/s (and query*segment pairs/s,
% of the FP64 pipe roofline).  Workload: BASELINE configs[4] = C5, the largest
single-GPU config (20,000 synthetic B-Rep faces, 64x64 uv grid per face =
81.92M queries, degree 1-5 rational Bezier p-curves, 30% periodic in u),
seeded synthetic data (wn_workloads.configs.gen_c5; the paper's datasets are not
in the container).  One STEP = one pass of the whole hot path over the batch:
wn_build_faces (segment prep K1, lifting K2a, planning, emission K2c) +
wn_query (bucketing K4 + query kernel K3) + wn_free_faces, inputs resident in
HBM.  Inputs (1.64 GB of queries) are larger than L2, so no flush is needed.

N > 1 (torchrun): weak scaling, every rank runs its own independent C5 batch
(seed 5 + rank); no data-path collective; the timed region is
bracketed by barriers and the max over ranks is reported.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed as it
stands on the host cores, each step a bounded sample of the same workload.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "winding-number queries/sec and query·segment pairs/sec; % of FP64 pipe peak"
UNIT = "queries/s"
WORKLOAD = ("C5 synthetic B-Rep batch / tessellation: 20000 faces, loops 1-8 (geometric), "
            "segments/loop 4-128 (log-uniform), degree 1-5 rational Bezier, 30% periodic in u, "
            "64x64 uv grid per face (81,920,000 queries), fp64")

# Roofline of the query kernel (DESIGN.md 6 "Roofline and algorithmic work"):
# ALGORITHMIC work = SURVEY 8(d)'s per-unit FP64-pipe instruction costs of the
# paper's literal Alg. 1 (the work the method as printed performs for the
# tests this run made) x the live unit counts of the same workload, divided by
# the kernel's CUDA-event time and by the FP64 pipe peak MEASURED in this run
# (wn_measure_fp_peak: DFMA chains, lane instructions / s).  Unit costs:
U_PRUNE = 71   # pruned (query, record) test: two distances, ellipse test, atan2 chord
U_TEST = 26    # test without a chord: hard root test, hierarchy node that descends, recursion node
U_EVAL = 22    # midpoint evaluation, 3 (n + 1) + 10 at the mean degree n = 3
U_LEAF = 45    # recursion leaf: chord + atan2


def algorithmic_work(cnt):
    """(phase-1 work, phase-2 work) in FP64-pipe lane instructions from the
    device counters (wn_get_counters) of one query launch."""
    span_pruned = cnt["span_tests"] - cnt["span_descended"]
    w1 = U_PRUNE * (cnt["seg_pruned"] + span_pruned) + U_TEST * (cnt["hard_pairs"] + cnt["span_descended"])
    w2 = U_TEST * cnt["nodes"] + U_EVAL * cnt["evals"] + U_LEAF * cnt["leaves"]
    return float(w1), float(w2)


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def max_over_ranks(x, dist=None, device=None):
    """Max of a per-rank scalar over all ranks (the timing rule: device time,
    max over ranks).  dist=None -> single process."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_seed(rank):
    """Weak scaling: every rank runs its own independent C5 batch."""
    return 5 + int(rank)


def _clock_sampler(gpu_index):
    cmd = ["nvidia-smi", "-i", str(gpu_index),
           "--query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
           "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
           "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
           "--format=csv,noheader,nounits", "-lms", "50"]
    try:
        return subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except OSError:
        return None


def _clock_summary(proc, t0, t1):
    if proc is None:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
    proc.terminate()
    try:
        out, _ = proc.communicate(timeout=5)
    except Exception:
        proc.kill()
        out = ""
    rows = []
    for line in out.strip().splitlines():
        parts = [p.strip() for p in line.split(",")]
        if len(parts) < 9:
            continue
        try:
            ts = time.mktime(time.strptime(parts[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
            rows.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
        except Exception:
            continue
    inwin = [r for r in rows if t0 - 1.0 <= r[0] <= t1 + 1.0] or rows
    if not inwin:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = sorted({names[i] for r in inwin for i, v in enumerate(r[3]) if v.lower() == "active"})
    return {"sm_mhz": statistics.median(r[1] for r in inwin), "sm_max_mhz": max(r[2] for r in inwin),
            "reasons": reasons, "samples": len(inwin)}


def _oracle_rate(wl, rng, cores, nq):
    """Per-query cost of the oracle from two pilots (fixed cost = its own
    lifting/pairing of all faces, paid once per call)."""
    import oracle
    ts = []
    for m in (512, 4096):
        idx = rng.choice(nq, size=min(nq, m), replace=False)
        t = time.perf_counter()
        oracle.query(wl, face_id=wl["face_id"][idx], uv=wl["uv"][idx], nthreads=cores)
        ts.append((len(idx), time.perf_counter() - t))
    (m0, t0), (m1, t1) = ts
    per_q = max((t1 - t0) / max(m1 - m0, 1), 1e-9)
    return per_q, max(t0 - per_q * m0, 0.0)


def _cpu_baseline(wl, target_s, rank_seed=0, one_thread_frac=0.0):
    """Oracle (as it stands) on a bounded random sample of the same workload."""
    import oracle
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(1234 + rank_seed)
    nq = len(wl["face_id"])
    per_q, fixed = _oracle_rate(wl, rng, cores, nq)
    m = int(min(nq, max(512, (target_s - fixed) / per_q)))
    idx = np.sort(rng.choice(nq, size=m, replace=False))
    t = time.perf_counter()
    oracle.query(wl, face_id=wl["face_id"][idx], uv=wl["uv"][idx], nthreads=cores)
    dt = time.perf_counter() - t
    out = {"value": m / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
           "sample": "%d random queries of the C5 batch (all faces eligible), one oracle call incl. its "
                     "own lifting/pairing of all faces, %.1f s wall" % (m, dt)}
    if one_thread_frac > 0:
        # fixed subsample (every k-th query) on ONE thread: the paper's single-threaded C++ 
        k = max(1, int(round(1.0 / one_thread_frac)))
        idx1 = np.arange(0, nq, k)
        t = time.perf_counter()
        oracle.query(wl, face_id=wl["face_id"][idx1], uv=wl["uv"][idx1], nthreads=1)
        d1 = time.perf_counter() - t
        out["single_thread"] = {"value": len(idx1) / d1, "unit": UNIT, "threads": 1,
                                "sample": "fixed %.2f%% subsample (every %d-th query of C5, %d queries), %.1f s wall"
                                          % (100.0 / k, k, len(idx1), d1)}
    return out, dt



def config_rates(wn, wl, precision, dev, st, fp64_peak, fp32_peak, nrep=10):
    """Build + query timing of one (smaller) BASELINE config on the device, its
    counters and its algorithmic roofline fraction (FP32 peak for fp32)."""
    import torch
    from wn_workloads import configs as G
    nq = len(wl["face_id"])
    T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    geo = [T(wl["ctrl_uv"], torch.float64), T(wl["ctrl_w"], torch.float64) if wl["ctrl_w"] is not None else None,
           T(wl["seg_degree"], torch.int32), T(wl["loop_seg_off"], torch.int32), T(wl["face_loop_off"], torch.int32),
           T(wl["face_periodic"], torch.uint8), T(wl["face_domain"], torch.float64)]
    fid, uv = T(wl["face_id"], torch.int32), T(wl["uv"], torch.float64)
    wnd = torch.empty(nq, dtype=torch.float64, device=dev)
    flg = torch.empty(nq, dtype=torch.uint8, device=dev)

    def q(faces):
        faces.query_raw(nq, fid.data_ptr(), uv.data_ptr(), wnd.data_ptr(), flg.data_ptr(), st.cuda_stream)

    for _ in range(3):
        f = wn.Faces.build(*geo, precision=precision, device=dev)
        q(f)
        f.close()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(nrep):
        f = wn.Faces.build(*geo, precision=precision, device=dev)
        q(f)
        f.close()
    e1.record(st)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / nrep
    faces = wn.Faces.build(*geo, precision=precision, device=dev)
    q(faces)
    torch.cuda.synchronize()
    faces.set_timing(True)
    e0.record(st)
    for _ in range(nrep):
        q(faces)
    e1.record(st)
    torch.cuda.synchronize()
    q_ms = e0.elapsed_time(e1) / nrep
    k3_ms, p1_ms, k3_n = faces.timing()
    faces.set_timing(False)
    faces.set_counters(True)
    q(faces)
    cnt = faces.counters()
    faces.set_counters(False)
    faces.close()
    k3_avg, p1_avg = k3_ms / max(k3_n, 1), p1_ms / max(k3_n, 1)
    w1, w2 = algorithmic_work(cnt)
    peak = fp32_peak if precision else fp64_peak
    pairs = G.n_input_pairs(wl)
    return {"queries": nq, "precision": "fp32" if precision else "fp64", "step_ms": step_ms, "query_ms": q_ms,
            "queries_per_s": nq / (q_ms / 1e3), "pairs_per_s": pairs / (q_ms / 1e3),
            "k3_ms": k3_avg, "phase1_ms": p1_avg,
            "roofline_frac": (w1 + w2) / (k3_avg / 1e3) / peak if k3_avg > 0 else None,
            "roofline_peak": "measured %s pipe" % ("FP32" if precision else "FP64"),
            "counters": {k: cnt[k] for k in ("pairs_tested", "span_tests", "hard_pairs", "nodes", "warp_records")}}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def run_reference(args, rank, world):

    if rank != 0:
        return 0
    from wn_workloads import configs as G
    wl = G.gen_c5(seed=5)
    import oracle
    cores = os.cpu_count() or 1
    # size one step as a bounded sample (~ a few seconds per step)
    rng = np.random.default_rng(99)
    nq = len(wl["face_id"])
    per_q, fixed = _oracle_rate(wl, rng, cores, nq)
    per_step = int(max(512, min(nq, (args.ref_step_s - fixed) / per_q)))
    samples = [np.sort(rng.choice(nq, size=per_step, replace=False)) for _ in range(args.warmup + args.steps)]
    for i in range(args.warmup):
        oracle.query(wl, face_id=wl["face_id"][samples[i]], uv=wl["uv"][samples[i]], nthreads=cores)
    t0 = time.perf_counter()
    for i in range(args.warmup, args.warmup + args.steps):
        oracle.query(wl, face_id=wl["face_id"][samples[i]], uv=wl["uv"][samples[i]], nthreads=cores)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "sample_per_step": per_step},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
                             "sample": "%d random C5 queries per step, %d steps" % (per_step, args.steps)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _ncu_traffic():
    """DRAM bytes per k_phase1 launch (dram__bytes_read.sum + dram__bytes_write.sum) from the committed
    `ncu --set full` capture of the same workload (profiles/round2/k_phase1_traffic.json, written by
    scripts/ncu_traffic.py); None if the file is absent.  Only `traffic` comes from it -- every other
    roofline input is measured live."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "round2", "k_phase1_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return int(d["dram_read_bytes"] + d["dram_write_bytes"]), d.get("source", "profiles/round2/k_phase1_traffic.json")
    except (OSError, ValueError, KeyError):
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wn", choices=["wn", "reference"])
    ap.add_argument("--angle-mode", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1-C4 extra keys")
    ap.add_argument("--shard", default="none", choices=["none", "faces"],
                    help="N > 1: 'none' = weak scaling (a batch per GPU), 'faces' = strong scaling (one batch, face shards)")
    ap.add_argument("--cpu-1t-frac", type=float, default=0.01, help="fixed subsample of the 1-thread oracle rate")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=6.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "wn" and not os.environ.get("WN_BENCH_ALLOW_SHORT"):
        args.warmup = 3
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2510_25159_b200 as wn
    from wn_workloads import configs as G

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    if args.shard == "faces" and world > 1:
        # strong scaling (SURVEY 8(e) face shards): ONE C5 batch split into
        # contiguous face ranges balanced by (segments + 1) x queries
        from paper_2510_25159_b200 import shard
        full = G.gen_c5(seed=5)
        bounds = shard.partition(shard.face_costs(full["loop_seg_off"], full["face_loop_off"], full["face_id"]), world)
        f0, f1 = int(bounds[rank]), int(bounds[rank + 1])
        wl, _ = shard.sub_batch(full, f0, f1, take_invalid=(rank == 0))
        wl["meta"] = dict(grid=full["meta"]["grid"], grid_box=np.ascontiguousarray(full["meta"]["grid_box"][f0:f1]))
        job_nq, job_pairs, scaling = len(full["face_id"]), G.n_input_pairs(full), "strong"
        del full
    else:
        wl = G.gen_c5(seed=rank_seed(rank))
        job_nq, job_pairs, scaling = None, None, "weak"
    nq = len(wl["face_id"])
    pairs = G.n_input_pairs(wl)
    if job_nq is None:
        job_nq, job_pairs = nq * world, pairs * world
    st = torch.cuda.current_stream(dev)
    T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    geo_np = [wl["ctrl_uv"], wl["ctrl_w"], wl["seg_degree"], wl["loop_seg_off"], wl["face_loop_off"],
              wl["face_periodic"], wl["face_domain"]]
    geo_dt = [torch.float64, torch.float64, torch.int32, torch.int32, torch.int32, torch.uint8, torch.float64]
    geo = [T(a, d) for a, d in zip(geo_np, geo_dt)]
    fid = T(wl["face_id"], torch.int32)
    uv = T(wl["uv"], torch.float64)
    wnd = torch.empty(nq, dtype=torch.float64, device=dev)
    flg = torch.empty(nq, dtype=torch.uint8, device=dev)
    kw = dict(angle_mode=args.angle_mode, device=dev)

    launches = {"build": 0, "query": 0}

    def step(timing=False):
        faces = wn.Faces.build(*geo, **kw)
        launches["build"] = wn.last_build_launches()
        if timing:
            faces.set_timing(True)
        faces.query_raw(nq, fid.data_ptr(), uv.data_ptr(), wnd.data_ptr(), flg.data_ptr(), st.cuda_stream)
        launches["query"] = wn.last_query_launches()
        k3 = None
        if timing:
            k3 = faces
        else:
            faces.close()
        return k3

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K full steps ----
    clk = _clock_sampler(local) if rank == 0 else None
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    tw0 = time.time()
    e0.record(st)
    k3_ms, p1_ms, k3_n = 0.0, 0.0, 0
    wn.freed_timing()              # drop stale entries
    for _ in range(args.steps):
        h = step(timing=True)     # K3 events recorded on the stream; no host wait per step
        h.close()
    e1.record(st)
    torch.cuda.synchronize()
    k3_ms, p1_ms, k3_n = wn.freed_timing()
    tw1 = time.time()
    if dist:
        dist.barrier()
    elapsed = e0.elapsed_time(e1)
    clocks = _clock_summary(clk, tw0, tw1) if rank == 0 else None
    t_max = max_over_ranks(elapsed, dist, dev)
    ms_step = t_max / args.steps
    value = job_nq / (ms_step / 1e3)
    pairs_s = job_pairs / (ms_step / 1e3)
    gpu_launches = (launches["build"] + launches["query"]) * args.steps

    # ---- query-only breakdown (untimed for the contract) ----
    faces = wn.Faces.build(*geo, **kw)
    for _ in range(2):
        faces.query_raw(nq, fid.data_ptr(), uv.data_ptr(), wnd.data_ptr(), flg.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    q0 = torch.cuda.Event(enable_timing=True)
    q1 = torch.cuda.Event(enable_timing=True)
    q0.record(st)
    nrep = 10
    for _ in range(nrep):
        faces.query_raw(nq, fid.data_ptr(), uv.data_ptr(), wnd.data_ptr(), flg.data_ptr(), st.cuda_stream)
    q1.record(st)
    torch.cuda.synchronize()
    q_ms = q0.elapsed_time(q1) / nrep
    faces.set_counters(True)
    faces.query_raw(nq, fid.data_ptr(), uv.data_ptr(), wnd.data_ptr(), flg.data_ptr(), st.cuda_stream)
    cnt = faces.counters()
    faces.set_counters(False)
    info = faces.info()
    flags = np.bincount(flg.cpu().numpy(), minlength=4).tolist()
    faces.close()

    # ---- e2e: public API with HOST buffers, copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        h_geo = [pin(a) for a in geo_np]
        h_fid = pin(wl["face_id"])
        h_uv = pin(wl["uv"])
        h_w = torch.empty(nq, dtype=torch.float64).pin_memory()
        h_f = torch.empty(nq, dtype=torch.uint8).pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in h_geo) + h_fid.numel() * 4 + h_uv.numel() * 8
        d2h = nq * 9

        def e2e_step():
            # geometry to the device, build, then the streamed host query
            # (wn_query_host: chunked copies in / kernels / copies out overlap)
            g = [t.to(dev, non_blocking=True) for t in h_geo]
            fc = wn.Faces.build(*g, **kw)
            fc.query_host(h_fid, h_uv, out=(h_w, h_f), sync=False)
            torch.cuda.current_stream(dev).synchronize()
            fc.close()

        e2e_step()
        ksteps = max(3, min(args.steps, 10))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(ksteps):
            e2e_step()
        b.record(st)
        torch.cuda.synchronize()
        et = max_over_ranks(a.elapsed_time(b), dist, dev)
        e2e = {"value": job_nq / (et / ksteps / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": ksteps, "ms_per_step": et / ksteps}

        # the same with the classification as the only result read back (h_winding = NULL)
        def e2e_flags_step():
            g = [t.to(dev, non_blocking=True) for t in h_geo]
            fc = wn.Faces.build(*g, **kw)
            fc.query_host(h_fid, h_uv, out=(None, h_f), sync=False, winding=False)
            torch.cuda.current_stream(dev).synchronize()
            fc.close()

        e2e_flags_step()
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(ksteps):
            e2e_flags_step()
        b.record(st)
        torch.cuda.synchronize()
        et = max_over_ranks(a.elapsed_time(b), dist, dev)
        e2e["flags_only"] = {"value": job_nq / (et / ksteps / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                             "d2h_bytes_per_step": int(nq), "ms_per_step": et / ksteps}

    # ---- implicit-grid path (wn_query_grid, Sec. 5.4.3 tessellation): the same
    # C5 cell-centred 64x64 grids, generated in the kernel (0 B/query in) ----
    ng_ = len(wl["meta"]["grid_box"])
    gn = wl["meta"]["grid"]
    gb = T(wl["meta"]["grid_box"], torch.float64)
    gface = torch.arange(ng_, dtype=torch.int32, device=dev)

    def gstep():
        fc = wn.Faces.build(*geo, **kw)
        fc.query_grid(gface, gb, gn, gn, out=(wnd, flg))
        fc.close()

    for _ in range(args.warmup):
        gstep()
    torch.cuda.synchronize()
    g0 = torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    g0.record(st)
    for _ in range(args.steps):
        gstep()
    g1.record(st)
    torch.cuda.synchronize()
    g_ms = max_over_ranks(g0.elapsed_time(g1), dist, dev) / args.steps
    fc = wn.Faces.build(*geo, **kw)
    fc.query_grid(gface, gb, gn, gn, out=(wnd, flg))
    torch.cuda.synchronize()
    g0.record(st)
    for _ in range(nrep):
        fc.query_grid(gface, gb, gn, gn, out=(wnd, flg))
    g1.record(st)
    torch.cuda.synchronize()
    gq_ms = g0.elapsed_time(g1) / nrep
    fc.close()
    grid = {"api": "wn_query_grid", "ms_per_step": g_ms, "value": job_nq / (g_ms / 1e3), "unit": UNIT,
            "query_ms": gq_ms, "query_queries_per_s": nq / (gq_ms / 1e3), "steps": args.steps,
            "input_bytes_per_query": 0, "e2e": None}
    if not args.no_e2e:
        h_gb = pin(wl["meta"]["grid_box"])
        side = torch.cuda.Stream(dev)
        nch = 8
        cg = (ng_ + nch - 1) // nch
        gq = gn * gn

        def grid_e2e_step(copy_w=True):
            g = [t.to(dev, non_blocking=True) for t in h_geo]
            b = h_gb.to(dev, non_blocking=True)
            fc = wn.Faces.build(*g, **kw)
            for c in range(nch):
                lo, hi = c * cg, min(ng_, (c + 1) * cg)
                if lo >= hi:
                    break
                fc.query_grid(gface[lo:hi], b[lo:hi], gn, gn, out=(wnd[lo * gq:hi * gq], flg[lo * gq:hi * gq]))
                ev = torch.cuda.Event()
                ev.record(st)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    if copy_w:
                        h_w[lo * gq:hi * gq].copy_(wnd[lo * gq:hi * gq], non_blocking=True)
                    h_f[lo * gq:hi * gq].copy_(flg[lo * gq:hi * gq], non_blocking=True)
            st.wait_stream(side)
            torch.cuda.current_stream(dev).synchronize()
            fc.close()

        grid_e2e_step()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(ksteps):
            grid_e2e_step()
        b.record(st)
        torch.cuda.synchronize()
        et = max_over_ranks(a.elapsed_time(b), dist, dev)
        grid["e2e"] = {"value": job_nq / (et / ksteps / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in h_geo) + h_gb.numel() * 8),
                       "d2h_bytes_per_step": int(d2h), "steps": ksteps, "ms_per_step": et / ksteps}
        grid_e2e_step(False)
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(ksteps):
            grid_e2e_step(False)
        b.record(st)
        torch.cuda.synchronize()
        et = max_over_ranks(a.elapsed_time(b), dist, dev)
        grid["e2e"]["flags_only"] = {"value": job_nq / (et / ksteps / 1e3), "unit": UNIT,
                                     "h2d_bytes_per_step": grid["e2e"]["h2d_bytes_per_step"],
                                     "d2h_bytes_per_step": int(nq), "ms_per_step": et / ksteps}

    # ---- roofline of the query kernel (algorithmic work / live time / measured peak) ----
    k3_avg = k3_ms / max(k3_n, 1)      # K3 (phase 1 + hard pairs + overflow + finish), CUDA events on the stream
    p1_avg = p1_ms / max(k3_n, 1)      # k_phase1 alone, same events, timed region
    fp64_peak, fp64_mhz = wn.measure_fp_peak(False, 0.05)
    fp32_peak, fp32_mhz = wn.measure_fp_peak(True, 0.05)
    w1, w2 = algorithmic_work(cnt)
    ach1 = w1 / (p1_avg / 1e3) / 1e9
    ach3 = (w1 + w2) / (k3_avg / 1e3) / 1e9
    lane_tests = cnt["pairs_tested"] + cnt["span_tests"]
    traffic, traffic_src = _ncu_traffic()
    roofline = {"bound": "alu", "achieved": ach1, "peak": fp64_peak / 1e9, "unit": "G FP64-pipe lane-inst/s",
                "frac": ach1 / (fp64_peak / 1e9), "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "wn::k_phase1<double>", "kernel_ms": p1_avg, "kernel_share_of_step": p1_avg / ms_step,
                "peak_source": "measured in this run: wn_measure_fp_peak (DFMA chains, lane inst/s) at %.0f MHz"
                               % fp64_mhz,
                "work": "SURVEY 8(d) unit costs x live counters: %d x pruned tests (seg %d + span %d) + %d x "
                        "(hard root tests %d + descending span tests %d)" % (
                            U_PRUNE, cnt["seg_pruned"], cnt["span_tests"] - cnt["span_descended"], U_TEST,
                            cnt["hard_pairs"], cnt["span_descended"]),
                "algorithmic_inst_per_launch": w1,
                "k3": {"ms": k3_avg, "achieved": ach3, "frac": ach3 / (fp64_peak / 1e9),
                       "algorithmic_inst_per_launch": w1 + w2,
                       "phase2": "%d x nodes %d + %d x evals %d + %d x leaves %d" % (
                           U_TEST, cnt["nodes"], U_EVAL, cnt["evals"], U_LEAF, cnt["leaves"])},
                "units": {"warp_records": cnt["warp_records"], "lane_tests": lane_tests,
                          "lane_utilisation": lane_tests / max(32 * cnt["warp_records"], 1),
                          "hbm_bytes_algorithmic": 29 * nq,
                          "hbm_gbs_algorithmic": 29 * nq / (p1_avg / 1e3) / 1e9},
                "peaks_measured": {"fp64_lane_fma_per_s": fp64_peak, "fp64_sm_mhz": fp64_mhz,
                                   "fp32_lane_fma_per_s": fp32_peak, "fp32_sm_mhz": fp32_mhz}}

    # ---- the other BASELINE configs (parity-test cases, reported as extra keys) ----
    others = None
    if rank == 0 and not args.no_configs:
        others = {}
        for name, gen, prec in (("C1", G.gen_c1, 0), ("C2", G.gen_c2, 0), ("C3", G.gen_c3, 0), ("C4", G.gen_c4, 0),
                                ("C4-fp32", lambda: G.to_fp32_inputs(G.gen_c4()), 1)):
            others[name] = config_rates(wn, gen(), prec, dev, st, fp64_peak, fp32_peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = _cpu_baseline(wl, args.cpu_seconds, one_thread_frac=args.cpu_1t_frac)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, no datasets)",
                "config": {"workload": WORKLOAD, "queries": nq, "input_segment_pairs": pairs,
                           "parallelism": ("single GPU" if world == 1 else "independent batch per GPU" if scaling == "weak"
                                           else "face shards of one batch (no exchange)"),
                           "l2": "inputs larger than L2 (1.64 GB queries per step), no flush",
                           "step": "wn_build_faces + wn_query + wn_free_faces",
                           "angle_mode": args.angle_mode},
                "pairs_per_s": pairs_s,
                "query_only": {"ms": q_ms, "queries_per_s": nq / (q_ms / 1e3), "pairs_per_s": pairs / (q_ms / 1e3)},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
                "grid": grid, "configs": others,
                "clocks": clocks, "counters": cnt, "faces_info": info, "flags": flags}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg /
`--impl reference` may import this package.  The product path
(paper_2510_25159_b200/) never imports it and shares no code with it.

The arithmetic lives in oracle/wn_oracle.c (plain C99 + OpenMP, fp64, no
FMA contraction); this file only compiles it with gcc and marshals numpy
arrays through ctypes.  See the header of wn_oracle.c for what is computed
and which PAPER.md passages each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile the oracle with gcc -O2 (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off",
                               "-fno-fast-math", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        u8 = C.POINTER(C.c_uint8)
        i64p = C.POINTER(C.c_int64)
        L.orc_chord.restype = C.c_double
        L.orc_chord.argtypes = [C.c_double] * 6
        L.orc_eval.argtypes = [C.c_int, dp, dp, C.c_double, dp]
        L.orc_deriv.argtypes = [C.c_int, dp, dp, C.c_double, dp]
        L.orc_segment_winding.argtypes = [C.c_int, dp, dp, C.c_double, C.c_double, C.c_double, dp]
        geo = [C.c_int, C.c_int, C.c_int, dp, dp, ip, ip, ip, u8, dp]
        L.orc_lift.restype = C.c_int
        L.orc_lift.argtypes = geo + [ip, ip, dp]
        L.orc_pairs.restype = C.c_int
        L.orc_pairs.argtypes = geo + [C.c_int, ip, ip, ip]
        L.orc_nurbs_decompose.restype = C.c_int
        L.orc_nurbs_decompose.argtypes = [C.c_int, C.c_int, dp, dp, dp, C.c_int, dp, dp]
        L.orc_query.restype = C.c_int
        L.orc_query.argtypes = geo + [C.c_int64, ip, dp, C.c_double, C.c_double, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.c_int, dp, u8, u8, dp, i64p, ip]
        _lib = L
    return _lib


def _p(a, ct):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))


def _geo(wl):
    ctrl = np.ascontiguousarray(wl["ctrl_uv"], dtype=np.float64)
    w = wl.get("ctrl_w")
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    deg = np.ascontiguousarray(wl["seg_degree"], dtype=np.int32)
    lo = np.ascontiguousarray(wl["loop_seg_off"], dtype=np.int32)
    fo = np.ascontiguousarray(wl["face_loop_off"], dtype=np.int32)
    per = np.ascontiguousarray(wl["face_periodic"], dtype=np.uint8)
    dom = np.ascontiguousarray(wl["face_domain"], dtype=np.float64).reshape(-1, 4)
    keep = (ctrl, w, deg, lo, fo, per, dom)
    args = [len(fo) - 1, len(lo) - 1, len(deg), _p(ctrl, C.c_double), _p(w, C.c_double),
            _p(deg, C.c_int), _p(lo, C.c_int), _p(fo, C.c_int), _p(per, C.c_uint8), _p(dom, C.c_double)]
    return args, keep


def chord(p, a, b):
    return lib().orc_chord(float(p[0]), float(p[1]), float(a[0]), float(a[1]), float(b[0]), float(b[1]))


def evaluate(P, w, t):
    P = np.ascontiguousarray(P, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(2)
    lib().orc_eval(P.shape[0] - 1, _p(P, C.c_double), _p(w, C.c_double), float(t), _p(out, C.c_double))
    return out


def derivative(P, w, t):
    P = np.ascontiguousarray(P, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(2)
    lib().orc_deriv(P.shape[0] - 1, _p(P, C.c_double), _p(w, C.c_double), float(t), _p(out, C.c_double))
    return out


def segment_winding(P, w, p, delta=1e-9):
    """(omega, near, dist_lb, pieces) of one segment about p."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(4)
    lib().orc_segment_winding(P.shape[0] - 1, _p(P, C.c_double), _p(w, C.c_double), float(p[0]),
                              float(p[1]), float(delta), _p(out, C.c_double))
    return out[0], bool(out[1]), out[2], int(out[3])


def lift(wl):
    """Oracle lifting: per-segment shifts [n_segs,2], per-loop class [n_loops,2], bbox [n_loops,4]."""
    args, keep = _geo(wl)
    ns, nl = args[2], args[1]
    sh = np.zeros((ns, 2), dtype=np.int32)
    cl = np.zeros((nl, 2), dtype=np.int32)
    bb = np.zeros((nl, 4))
    rc = lib().orc_lift(*args, _p(sh, C.c_int), _p(cl, C.c_int), _p(bb, C.c_double))
    if rc != 0:
        raise ValueError("oracle lift: invalid geometry rc=%d" % rc)
    return sh, cl, bb


def pairs(wl, N5=8):
    args, keep = _geo(wl)
    nl, nf = args[1], args[0]
    pr = np.zeros(nl, dtype=np.int32)
    ps = np.zeros((nl, 2), dtype=np.int32)
    fe = np.zeros(nf, dtype=np.int32)
    rc = lib().orc_pairs(*args, int(N5), _p(pr, C.c_int), _p(ps, C.c_int), _p(fe, C.c_int))
    if rc != 0:
        raise ValueError("oracle pairs: invalid geometry rc=%d" % rc)
    return pr, ps, fe


def query(wl, face_id=None, uv=None, delta=1e-9, tol=1e-9, N5=8, rule=0, reduce=True, strict=True, nthreads=0):
    """Oracle winding numbers for a batch.  Returns dict(w, flag, comparable,
    dist_lb, pieces, face_err)."""
    args, keep = _geo(wl)
    fid = np.ascontiguousarray(wl["face_id"] if face_id is None else face_id, dtype=np.int32)
    q = np.ascontiguousarray(wl["uv"] if uv is None else uv, dtype=np.float64).reshape(-1, 2)
    nq = fid.shape[0]
    w = np.zeros(nq)
    fl = np.zeros(nq, dtype=np.uint8)
    cm = np.zeros(nq, dtype=np.uint8)
    dl = np.zeros(nq)
    pc = np.zeros(nq, dtype=np.int64)
    fe = np.zeros(args[0], dtype=np.int32)
    rc = lib().orc_query(*args, nq, _p(fid, C.c_int), _p(q, C.c_double), float(delta), float(tol),
                         int(N5), int(rule), int(bool(reduce)), int(bool(strict)), int(nthreads), _p(w, C.c_double),
                         _p(fl, C.c_uint8), _p(cm, C.c_uint8), _p(dl, C.c_double), _p(pc, C.c_int64),
                         _p(fe, C.c_int))
    if rc != 0:
        raise ValueError("oracle query: invalid geometry rc=%d" % rc)
    return dict(w=w, flag=fl, comparable=cm.astype(bool), dist_lb=dl, pieces=pc, face_err=fe)


def nurbs_decompose(p, P, w, U):
    """Oracle NURBS -> rational Bezier (repeated knot insertion).  Returns a list
    of (P [p+1,2], w [p+1]) segments."""
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(-1, 2)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    cap = len(U)
    oP = np.zeros((cap, p + 1, 2))
    ow = np.zeros((cap, p + 1))
    rc = lib().orc_nurbs_decompose(int(p), P.shape[0], _p(P, C.c_double), _p(w, C.c_double), _p(U, C.c_double),
                                   cap, _p(oP, C.c_double), _p(ow, C.c_double))
    if rc < 0:
        raise ValueError("oracle nurbs_decompose: rc=%d" % rc)
    return [(oP[i].copy(), ow[i].copy()) for i in range(rc)]


def nurbs_to_bezier_workload(wl):
    """The oracle's own Bezier form of a NURBS workload (wn_workloads.gen_nurbs
    layout): every curve decomposed by nurbs_decompose, loops re-indexed."""
    ctrl, wts, deg, lso = [], [], [], [0]
    co, ko, lco = wl["curve_ctrl_off"], wl["curve_knot_off"], wl["loop_curve_off"]
    for l in range(len(lco) - 1):
        nseg = 0
        for c in range(lco[l], lco[l + 1]):
            p = int(wl["curve_degree"][c])
            segs = nurbs_decompose(p, wl["ctrl_uv"][co[c]:co[c + 1]],
                                   None if wl["ctrl_w"] is None else wl["ctrl_w"][co[c]:co[c + 1]],
                                   wl["knots"][ko[c]:ko[c + 1]])
            for P, w in segs:
                ctrl.append(P)
                wts.append(w)
                deg.append(p)
            nseg += len(segs)
        lso.append(lso[-1] + nseg)
    out = dict(wl)
    out.update(ctrl_uv=np.ascontiguousarray(np.concatenate(ctrl)), ctrl_w=np.ascontiguousarray(np.concatenate(wts)),
               seg_degree=np.asarray(deg, dtype=np.int32), loop_seg_off=np.asarray(lso, dtype=np.int32))
    return out

"""paper_2510_25159_b200 -- B200-native batched generalized-winding-number
containment queries on trimmed faces (arXiv 2510.25159).

Thin ctypes binding over the C ABI in include/wn.h (libwn.so, built in-tree for
sm_100a).  This module only marshals arguments: every step of the path runs in
the CUDA kernels of libwn.  There is no CPU fallback: without the extension or
without a CUDA device every entry point raises.

    import paper_2510_25159_b200 as wn
    faces = wn.Faces.build(ctrl_uv, ctrl_w, seg_degree, loop_seg_off, face_loop_off,
                           face_periodic, face_domain)        # torch CUDA tensors or numpy
    winding, flag = faces.query(face_id, uv)                   # torch CUDA tensors
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("WN_LIB_OVERRIDE") or os.path.join(_HERE, "libwn.so")   # override: dev experiments only
_lib = None

WN_OK = 0
STATUS = {0: "WN_OK", 1: "WN_ERR_ARG", 2: "WN_ERR_GEOM", 3: "WN_ERR_TOPOLOGY", 4: "WN_ERR_CUDA",
          5: "WN_ERR_NOMEM", 6: "WN_ERR_UNSUPPORTED"}
FACE_STATUS = {0: "ok", 1: "B1", 2: "unbalanced", 3: "class", 4: "general_pq", 5: "pairing", 6: "geom"}
EXPORTS = ["wn_build_faces", "wn_query", "wn_faces_info", "wn_set_counters", "wn_get_counters",
           "wn_set_timing", "wn_get_timing", "wn_free_faces", "wn_last_error", "wn_last_query_launches",
           "wn_last_build_launches", "wn_segment_prep", "wn_trim_memory", "wn_query_host", "wn_query_grid",
           "wn_nurbs_to_bezier", "wn_build_faces_nurbs", "wn_measure_fp_peak",
           "wn_recursion_bounds"]
COUNTER_NAMES = ["pairs_tested", "hard_pairs", "nodes", "evals", "leaves", "max_depth",
                 "warp_skips", "on_boundary", "span_tests", "warp_records", "span_descended",
                 "seg_pruned"]


class WNError(RuntimeError):
    def __init__(self, status, msg, face_status=None):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status
        self.face_status = face_status


class Options(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_depth", C.c_int), ("precision", C.c_int),
                ("rule", C.c_int), ("angle_mode", C.c_int), ("strict", C.c_int), ("hierarchy", C.c_int)]


class FacesInfo(C.Structure):
    _fields_ = [("n_records", C.c_int64), ("n_seg_records", C.c_int64), ("n_groups", C.c_int64),
                ("n_lines", C.c_int64), ("bytes", C.c_int64), ("precision", C.c_int32),
                ("max_face_records", C.c_int32), ("n_copy_groups", C.c_int64), ("n_bands", C.c_int64)]


def lib_path():
    return _LIBPATH


def load():
    """Load libwn.so (build it first with `python -m paper_2510_25159_b200._build`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIBPATH):
            raise ImportError("libwn.so not built (run __graft_entry__.build() or "
                              "python -m paper_2510_25159_b200._build); there is no CPU fallback")
        L = C.CDLL(_LIBPATH)
        vp = C.c_void_p
        L.wn_build_faces.restype = C.c_int
        L.wn_build_faces.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp, vp,
                                     C.POINTER(Options), vp, C.POINTER(vp), vp]
        L.wn_query.restype = C.c_int
        L.wn_query.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp]
        L.wn_query_host.restype = C.c_int
        L.wn_query_host.argtypes = [vp, C.c_int64, vp, vp, vp, vp, C.c_int64, vp]
        L.wn_query_grid.restype = C.c_int
        L.wn_nurbs_to_bezier.restype = C.c_int
        L.wn_nurbs_to_bezier.argtypes = [C.c_int32] * 3 + [vp] * 6 + [C.c_int32, C.c_int32] + [vp] * 7
        L.wn_build_faces_nurbs.restype = C.c_int
        L.wn_build_faces_nurbs.argtypes = [C.c_int32] * 5 + [vp] * 10 + [vp, vp, vp, vp]
        L.wn_query_grid.argtypes = [vp, C.c_int32, vp, vp, C.c_int32, C.c_int32, vp, vp, vp]
        L.wn_faces_info.restype = C.c_int
        L.wn_faces_info.argtypes = [vp, C.POINTER(FacesInfo)]
        L.wn_set_counters.restype = C.c_int
        L.wn_set_counters.argtypes = [vp, C.c_int]
        L.wn_get_counters.restype = C.c_int
        L.wn_get_counters.argtypes = [vp, vp, C.POINTER(C.c_int64)]
        L.wn_set_timing.restype = C.c_int
        L.wn_set_timing.argtypes = [vp, C.c_int]
        L.wn_get_timing.restype = C.c_int
        L.wn_get_timing.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.wn_last_build_launches.restype = C.c_int32
        L.wn_last_build_launches.argtypes = []
        L.wn_segment_prep.restype = C.c_int
        L.wn_segment_prep.argtypes = [C.c_int32, vp, vp, vp, vp, vp]
        L.wn_trim_memory.restype = None
        L.wn_trim_memory.argtypes = []
        L.wn_free_faces.restype = None
        L.wn_free_faces.argtypes = [vp]
        L.wn_last_error.restype = C.c_char_p
        L.wn_last_error.argtypes = []
        L.wn_recursion_bounds.restype = C.c_int
        L.wn_recursion_bounds.argtypes = [vp, vp, vp]
        L.wn_measure_fp_peak.restype = C.c_int
        L.wn_measure_fp_peak.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.wn_last_query_launches.restype = C.c_int32
        L.wn_last_query_launches.argtypes = []
        _lib = L
    return _lib


def last_error():
    return load().wn_last_error().decode()


def _torch():
    import torch
    return torch


def _dev(x, dtype, device):
    """numpy / torch -> contiguous CUDA tensor of dtype (marshalling only)."""
    torch = _torch()
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device=device, dtype=dtype).contiguous()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream, device):
    torch = _torch()
    s = torch.cuda.current_stream(device) if stream is None else stream
    return C.c_void_p(s.cuda_stream)


@dataclass
class QueryResult:
    winding: "object"
    flag: "object"


class Faces:
    """A built face set (owns the device records of libwn)."""

    def __init__(self, handle, device, n_faces, options):
        self._h = handle
        self.device = device
        self.n_faces = n_faces
        self.options = options

    @classmethod
    def build(cls, ctrl_uv, ctrl_w, seg_degree, loop_seg_off, face_loop_off, face_periodic,
              face_domain, eps=0.0, max_depth=0, precision=0, rule=0, angle_mode=0, strict=True,
              hierarchy=True, device=None, stream=None):
        torch = _torch()
        L = load()
        if not torch.cuda.is_available():
            raise WNError(4, "no CUDA device (libwn has no CPU fallback)")
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        ctrl = _dev(ctrl_uv, torch.float64, device).reshape(-1, 2)
        w = _dev(ctrl_w, torch.float64, device)
        deg = _dev(seg_degree, torch.int32, device)
        lso = _dev(loop_seg_off, torch.int32, device)
        flo = _dev(face_loop_off, torch.int32, device)
        per = _dev(face_periodic, torch.uint8, device)
        dom = _dev(face_domain, torch.float64, device).reshape(-1, 4)
        nf, nl, ns = flo.numel() - 1, lso.numel() - 1, deg.numel()
        status = torch.zeros(max(nf, 1), dtype=torch.int32, device=device)
        opts = Options(float(eps), int(max_depth), int(precision), int(rule), int(angle_mode), int(bool(strict)),
                       int(bool(hierarchy)))
        h = C.c_void_p()
        with torch.cuda.device(device):
            rc = L.wn_build_faces(nf, nl, ns, _ptr(ctrl), _ptr(w), _ptr(deg), _ptr(lso), _ptr(flo),
                                  _ptr(per), _ptr(dom), C.byref(opts), _stream(stream, device), C.byref(h),
                                  _ptr(status))
        if rc != WN_OK:
            raise WNError(rc, last_error(), status[:nf].cpu().numpy())
        if stream is not None and hasattr(stream, "cuda_stream"):
            # the build is asynchronous on `stream`: keep the inputs alive on it
            for t in (ctrl, w, deg, lso, flo, per, dom, status):
                if t is not None and t.is_cuda:
                    t.record_stream(stream)
        return cls(h, device, nf, opts)

    @classmethod
    def build_nurbs(cls, ctrl_uv, ctrl_w, curve_degree, curve_ctrl_off, knots, curve_knot_off, loop_curve_off,
                    face_loop_off, face_periodic, face_domain, eps=0.0, max_depth=0, precision=0, rule=0,
                    angle_mode=0, strict=True, hierarchy=True, device=None, stream=None):
        """wn_build_faces_nurbs: faces bounded by loops of clamped NURBS curves
        (decomposed into rational Bezier segments on the device)."""
        torch = _torch()
        L = load()
        if not torch.cuda.is_available():
            raise WNError(4, "no CUDA device (libwn has no CPU fallback)")
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        ctrl = _dev(ctrl_uv, torch.float64, device).reshape(-1, 2)
        w = _dev(ctrl_w, torch.float64, device)
        deg = _dev(curve_degree, torch.int32, device)
        co = _dev(curve_ctrl_off, torch.int32, device)
        kn = _dev(knots, torch.float64, device)
        ko = _dev(curve_knot_off, torch.int32, device)
        lco = _dev(loop_curve_off, torch.int32, device)
        flo = _dev(face_loop_off, torch.int32, device)
        per = _dev(face_periodic, torch.uint8, device)
        dom = _dev(face_domain, torch.float64, device).reshape(-1, 4)
        nf, nl, nc = flo.numel() - 1, lco.numel() - 1, deg.numel()
        status = torch.zeros(max(nf, 1), dtype=torch.int32, device=device)
        opts = Options(float(eps), int(max_depth), int(precision), int(rule), int(angle_mode), int(bool(strict)),
                       int(bool(hierarchy)))
        h = C.c_void_p()
        with torch.cuda.device(device):
            rc = L.wn_build_faces_nurbs(nf, nl, nc, ctrl.shape[0], kn.numel(), _ptr(ctrl), _ptr(w), _ptr(deg),
                                        _ptr(co), _ptr(kn), _ptr(ko), _ptr(lco), _ptr(flo), _ptr(per), _ptr(dom),
                                        C.byref(opts), _stream(stream, device), C.byref(h), _ptr(status))
        if rc != WN_OK:
            raise WNError(rc, last_error(), status[:nf].cpu().numpy())
        if stream is not None and hasattr(stream, "cuda_stream"):
            for t in (ctrl, w, deg, co, kn, ko, lco, flo, per, dom, status):
                if t is not None and t.is_cuda:
                    t.record_stream(stream)
        return cls(h, device, nf, opts)

    @classmethod
    def from_nurbs_workload(cls, wl, **kw):
        return cls.build_nurbs(wl["ctrl_uv"], wl["ctrl_w"], wl["curve_degree"], wl["curve_ctrl_off"], wl["knots"],
                               wl["curve_knot_off"], wl["loop_curve_off"], wl["face_loop_off"],
                               wl["face_periodic"], wl["face_domain"], **kw)

    @classmethod
    def from_workload(cls, wl, **kw):
        return cls.build(wl["ctrl_uv"], wl["ctrl_w"], wl["seg_degree"], wl["loop_seg_off"],
                         wl["face_loop_off"], wl["face_periodic"], wl["face_domain"], **kw)

    def query(self, face_id, uv, out=None, stream=None):
        """(winding float64 [n], flag uint8 [n]) as CUDA tensors; asynchronous on `stream`."""
        torch = _torch()
        fid = _dev(face_id, torch.int32, self.device)
        q = _dev(uv, torch.float64, self.device).reshape(-1, 2)
        n = fid.numel()
        if out is None:
            wnd = torch.empty(n, dtype=torch.float64, device=self.device)
            flg = torch.empty(n, dtype=torch.uint8, device=self.device)
        else:
            wnd, flg = out
        with torch.cuda.device(self.device):
            rc = load().wn_query(self._h, n, _ptr(fid), _ptr(q), _ptr(wnd), _ptr(flg),
                                 _stream(stream, self.device))
        if rc != WN_OK:
            raise WNError(rc, last_error())
        return QueryResult(wnd, flg)

    def query_grid(self, grid_face, grid_box, nu, nv, out=None, stream=None):
        """Implicit-grid query (wn_query_grid): nu x nv cell centres of each box
        grid_box[g] = (u_lo, v_lo, u_hi, v_hi) of face grid_face[g]; returns
        (winding float64 [n_grid*nv*nu], flag uint8 [...]) as CUDA tensors, row
        major per grid (v outer, u inner); asynchronous on `stream`."""
        torch = _torch()
        gf = _dev(grid_face, torch.int32, self.device)
        gb = _dev(grid_box, torch.float64, self.device).reshape(-1, 4)
        ng = gf.numel()
        n = ng * int(nu) * int(nv)
        if out is None:
            wnd = torch.empty(n, dtype=torch.float64, device=self.device)
            flg = torch.empty(n, dtype=torch.uint8, device=self.device)
        else:
            wnd, flg = out
        with torch.cuda.device(self.device):
            rc = load().wn_query_grid(self._h, ng, _ptr(gf), _ptr(gb), int(nu), int(nv), _ptr(wnd), _ptr(flg),
                                      _stream(stream, self.device))
        if rc != WN_OK:
            raise WNError(rc, last_error())
        if stream is not None and hasattr(stream, "cuda_stream"):
            gf.record_stream(stream)
            gb.record_stream(stream)
        self._keep_grid = (gf, gb)
        return QueryResult(wnd, flg)

    def query_host(self, face_id, uv, out=None, chunk=0, stream=None, sync=True, winding=True):
        """Streamed query of HOST arrays (wn_query_host): chunks are copied in,
        queried and copied back on overlapping streams.  face_id / uv: CPU
        tensors or numpy arrays (pinned CPU tensors give the overlap); returns
        (winding float64 [n], flag uint8 [n]) as CPU tensors, valid after the
        stream is synchronised (sync=True waits).  winding=False: only the flags
        come back (result.winding is None; out = (None, flag) or None)."""
        torch = _torch()

        def cpu(x, dt):
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
            if t.is_cuda:
                raise WNError(1, "query_host takes host arrays")
            return t.to(dt).contiguous()

        fid = cpu(face_id, torch.int32)
        q = cpu(uv, torch.float64).reshape(-1, 2)
        n = fid.numel()
        if out is None:
            pin = fid.is_pinned()
            wnd = torch.empty(n, dtype=torch.float64, pin_memory=pin) if winding else None
            flg = torch.empty(n, dtype=torch.uint8, pin_memory=pin)
        else:
            wnd, flg = out
            if not winding:
                wnd = None
        s = _stream(stream, self.device)
        with torch.cuda.device(self.device):
            rc = load().wn_query_host(self._h, n, C.c_void_p(fid.data_ptr()), C.c_void_p(q.data_ptr()),
                                      C.c_void_p(wnd.data_ptr() if wnd is not None else None),
                                      C.c_void_p(flg.data_ptr()), int(chunk), s)
        if rc != WN_OK:
            raise WNError(rc, last_error())
        if sync:
            torch.cuda.current_stream(self.device).synchronize() if stream is None else stream.synchronize()
        self._keep = (fid, q)   # inputs must outlive the asynchronous copies
        return QueryResult(wnd, flg)

    def query_raw(self, n, face_id_ptr, uv_ptr, winding_ptr, flag_ptr, stream_handle):
        """Pointer-level call (already-resident buffers; used by bench.py)."""
        rc = load().wn_query(self._h, int(n), C.c_void_p(face_id_ptr), C.c_void_p(uv_ptr),
                             C.c_void_p(winding_ptr), C.c_void_p(flag_ptr), C.c_void_p(stream_handle))
        if rc != WN_OK:
            raise WNError(rc, last_error())

    def info(self):
        inf = FacesInfo()
        rc = load().wn_faces_info(self._h, C.byref(inf))
        if rc != WN_OK:
            raise WNError(rc, last_error())
        return {k: getattr(inf, k) for k, _ in FacesInfo._fields_}

    def recursion_bounds(self, n_segs):
        """[n_segs, 23] = (B, Bq[8], Sp[14]) per input segment (wn_recursion_bounds)."""
        torch = _torch()
        out = torch.empty((max(int(n_segs), 1), 23), dtype=torch.float64, device=self.device)
        rc = load().wn_recursion_bounds(self._h, _ptr(out), _stream(None, self.device))
        if rc != WN_OK:
            raise WNError(rc, last_error())
        return out[:n_segs]

    def set_counters(self, enable=True):
        load().wn_set_counters(self._h, int(bool(enable)))

    def counters(self, stream=None):
        arr = (C.c_int64 * 12)()
        rc = load().wn_get_counters(self._h, _stream(stream, self.device), arr)
        if rc != WN_OK:
            raise WNError(rc, last_error())
        return dict(zip(COUNTER_NAMES, list(arr)))

    def set_timing(self, enable=True):
        load().wn_set_timing(self._h, int(bool(enable)))

    def timing(self):
        """(summed K3 ms, summed phase-1 ms, timed queries) since the last call (waits on events)."""
        ms = C.c_double()
        p1 = C.c_double()
        n = C.c_int64()
        rc = load().wn_get_timing(self._h, C.byref(ms), C.byref(p1), C.byref(n))
        if rc != WN_OK:
            raise WNError(rc, last_error())
        return ms.value, p1.value, n.value

    def close(self):
        if self._h:
            load().wn_free_faces(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def freed_timing():
    """(K3 ms, phase-1 ms, timed queries) of handles freed before their timing was read."""
    ms = C.c_double()
    p1 = C.c_double()
    n = C.c_int64()
    rc = load().wn_get_timing(None, C.byref(ms), C.byref(p1), C.byref(n))
    if rc != WN_OK:
        raise WNError(rc, last_error())
    return ms.value, p1.value, n.value


def segment_prep(ctrl_uv, ctrl_w, seg_degree, device=None, stream=None):
    """K1 alone: [n_segs, 18] = (B, S0, Bq[8], Lq[8]) per segment (no margins)."""
    torch = _torch()
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    ctrl = _dev(ctrl_uv, torch.float64, device).reshape(-1, 2)
    w = _dev(ctrl_w, torch.float64, device)
    deg = _dev(seg_degree, torch.int32, device)
    out = torch.empty((deg.numel(), 18), dtype=torch.float64, device=device)
    rc = load().wn_segment_prep(deg.numel(), _ptr(ctrl), _ptr(w), _ptr(deg), _ptr(out), _stream(stream, device))
    if rc != WN_OK:
        raise WNError(rc, last_error())
    return out


def measure_fp_peak(fp32=False, seconds=0.05):
    """(lane FMA instructions / s, SM MHz during the run) of the device's FP64
    (fp32=False) or FP32 pipe: wn_measure_fp_peak."""
    r, m = C.c_double(), C.c_double()
    rc = load().wn_measure_fp_peak(int(bool(fp32)), float(seconds), C.byref(r), C.byref(m))
    if rc != WN_OK:
        raise WNError(rc, last_error())
    return r.value, m.value


def last_query_launches():
    return int(load().wn_last_query_launches())


def last_build_launches():
    return int(load().wn_last_build_launches())


def nurbs_to_bezier(ctrl_uv, ctrl_w, curve_degree, curve_ctrl_off, knots, curve_knot_off, device=None):
    """wn_nurbs_to_bezier on the device: returns (curve_seg_off, bez_uv, bez_w,
    bez_degree) as CUDA tensors (the wn_build_faces segment layout)."""
    torch = _torch()
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    ctrl = _dev(ctrl_uv, torch.float64, device).reshape(-1, 2)
    w = _dev(ctrl_w, torch.float64, device)
    deg = _dev(curve_degree, torch.int32, device)
    co = _dev(curve_ctrl_off, torch.int32, device)
    kn = _dev(knots, torch.float64, device)
    ko = _dev(curve_knot_off, torch.int32, device)
    nc = deg.numel()
    d = np.asarray(curve_degree, dtype=np.int64)
    nctrl = np.diff(np.asarray(curve_ctrl_off, dtype=np.int64))
    seg_cap = int(np.sum(np.maximum(nctrl - d, 0)))
    pt_cap = int(np.sum(np.maximum(nctrl - d, 0) * (d + 1)))
    cso = torch.empty(nc + 1, dtype=torch.int32, device=device)
    bz = torch.empty((max(pt_cap, 1), 2), dtype=torch.float64, device=device)
    bw = torch.empty(max(pt_cap, 1), dtype=torch.float64, device=device)
    bd = torch.empty(max(seg_cap, 1), dtype=torch.int32, device=device)
    ns, npt = C.c_int32(), C.c_int32()
    with torch.cuda.device(device):
        rc = load().wn_nurbs_to_bezier(nc, ctrl.shape[0], kn.numel(), _ptr(ctrl), _ptr(w), _ptr(deg), _ptr(co),
                                       _ptr(kn), _ptr(ko), seg_cap, pt_cap, _ptr(cso), _ptr(bz), _ptr(bw),
                                       _ptr(bd), C.byref(ns), C.byref(npt), _stream(None, device))
    if rc != WN_OK:
        raise WNError(rc, last_error())
    return cso, bz[:npt.value], bw[:npt.value], bd[:ns.value]

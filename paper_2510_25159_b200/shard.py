"""Face-shard partitioning of one batch across GPUs.

Queries are independent and faces are independent at build time, so a batch
shards with no exchange step: rank r builds only a contiguous range of faces
and answers only the queries on those faces.  The ranges are balanced by the
estimated cost of a face, (input segments + 1) x queries on the face -- the
number of (query, segment) pairs the method starts from (the O(n)
per-query work before pruning).  Host-side numpy only (argument marshalling
for the per-rank wn_build_faces / wn_query calls); every computation of the
path still runs in libwn on the rank's GPU.
"""
from __future__ import annotations

import numpy as np


def face_costs(loop_seg_off, face_loop_off, face_id, n_faces=None):
    """(input segments + 1) x queries per face."""
    lso = np.asarray(loop_seg_off, dtype=np.int64)
    flo = np.asarray(face_loop_off, dtype=np.int64)
    nf = len(flo) - 1 if n_faces is None else int(n_faces)
    segs = lso[flo[1:]] - lso[flo[:-1]]
    fid = np.asarray(face_id, dtype=np.int64)
    ok = (fid >= 0) & (fid < nf)
    q = np.bincount(fid[ok], minlength=nf).astype(np.int64)
    return (segs + 1) * q


def partition(costs, world):
    """Contiguous face ranges [bounds[r], bounds[r+1]) for r = 0..world-1 that
    balance the summed cost: rank r's range ends at the first face whose cost
    prefix reaches (r+1)/world of the total.  Every face in exactly one range;
    the heaviest range exceeds the mean by at most one face's cost."""
    c = np.asarray(costs, dtype=np.float64)
    nf = len(c)
    world = int(world)
    if world < 1:
        raise ValueError("world must be >= 1")
    pre = np.concatenate([[0.0], np.cumsum(c)])
    tot = pre[-1]
    bounds = [0]
    for r in range(1, world):
        b = int(np.searchsorted(pre, tot * r / world, side="left"))
        b = min(max(b, bounds[-1]), nf)
        bounds.append(b)
    bounds.append(nf)
    return np.asarray(bounds, dtype=np.int64)


def sub_batch(wl, f0, f1, take_invalid=False):
    """The sub-workload of faces [f0, f1) in the wn_build_faces layout (CSR
    rebased, face ids renumbered) and the original positions of its queries.
    take_invalid (rank 0): also the queries whose face id names no face (they
    keep an invalid id and get flag 3)."""
    lso = np.asarray(wl["loop_seg_off"], dtype=np.int64)
    flo = np.asarray(wl["face_loop_off"], dtype=np.int64)
    deg = np.asarray(wl["seg_degree"], dtype=np.int64)
    coff = np.concatenate([[0], np.cumsum(deg + 1)])
    l0, l1 = flo[f0], flo[f1]
    s0, s1 = lso[l0], lso[l1]
    c0, c1 = coff[s0], coff[s1]
    fid = np.asarray(wl["face_id"], dtype=np.int64)
    nf = len(flo) - 1
    mine = (fid >= f0) & (fid < f1)
    if take_invalid:
        mine |= (fid < 0) | (fid >= nf)
    qsel = np.nonzero(mine)[0]
    loc = fid[qsel] - f0
    loc[(fid[qsel] < f0) | (fid[qsel] >= f1)] = -1
    out = dict(
        ctrl_uv=np.ascontiguousarray(wl["ctrl_uv"][c0:c1]),
        ctrl_w=None if wl["ctrl_w"] is None else np.ascontiguousarray(wl["ctrl_w"][c0:c1]),
        seg_degree=np.ascontiguousarray(wl["seg_degree"][s0:s1]),
        loop_seg_off=np.ascontiguousarray((lso[l0:l1 + 1] - s0).astype(np.int32)),
        face_loop_off=np.ascontiguousarray((flo[f0:f1 + 1] - l0).astype(np.int32)),
        face_periodic=np.ascontiguousarray(wl["face_periodic"][f0:f1]),
        face_domain=np.ascontiguousarray(np.asarray(wl["face_domain"]).reshape(-1, 4)[f0:f1]),
        face_id=np.ascontiguousarray(loc.astype(np.int32)),
        uv=np.ascontiguousarray(np.asarray(wl["uv"]).reshape(-1, 2)[qsel]),
    )
    return out, qsel

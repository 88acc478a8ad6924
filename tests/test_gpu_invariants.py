"""Properties of the winding number that hold at any size, checked through the
C ABI on the GPU alone (-m gpu): no expected value comes from the oracle here.

* orientation reversal: omega(p, -gamma) = -omega(p, gamma) (Eq. 1, P:254-258:
  the integral changes sign with the direction of traversal);
* additivity over loops: a face holding the loops of A and of B
  has omega = omega_A + omega_B;
* exact scaling: multiplying every coordinate, period and eps by a power of two
  is exact in binary floating point, so every decision of Alg. 1
  repeats and flags AND winding numbers are bit-identical;
* two handles queried concurrently on two streams give the results of the
  sequential runs (no shared scratch between calls)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_25159_b200 as wn  # noqa: E402
from tests import helpers as H  # noqa: E402
from wn_workloads import configs as G  # noqa: E402


def _faces_of(wl):
    """[(loops, periodic, domain)] of a generated workload (stored coordinates)."""
    loops = H.loops_of(wl)
    flo = wl["face_loop_off"]
    return [([loops[l] for l in range(flo[f], flo[f + 1])], int(wl["face_periodic"][f]),
             tuple(wl["face_domain"][f])) for f in range(len(flo) - 1)]


def _query(wl, **kw):
    faces = wn.Faces.from_workload(wl, **kw)
    r = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    return w, fl


def _reverse(segs):
    return [(np.ascontiguousarray(P[::-1]), None if w is None else np.ascontiguousarray(w[::-1])) for P, w in segs[::-1]]


@pytest.mark.parametrize("gen", ["c2", "c5", "c5-generic"])
def test_orientation_reversal(gen):
    wl = {"c2": lambda: G.gen_c2(n_queries=100_000),
          "c5": lambda: G.gen_c5(n_faces=300, grid=24),
          "c5-generic": lambda: G.gen_c5(n_faces=200, grid=24, exact=False, store_jitter=2)}[gen]()
    w, fl = _query(wl)
    rev = H.make_wl([([_reverse(l) for l in loops], per, dom) for loops, per, dom in _faces_of(wl)],
                    wl["uv"], wl["face_id"])
    wr, flr = _query(rev)
    ok = (fl < 2) & (flr < 2)
    assert ok.mean() > 0.99
    assert np.array_equal(fl >= 2, flr >= 2)          # on-boundary / invalid decisions do not depend on the direction
    # closed loops: integers, exactly negated; generic periodic data: within the parity tolerance
    tol = 0.0 if gen != "c5-generic" else 1e-9
    assert np.max(np.abs(w[ok] + wr[ok])) <= tol
    assert np.array_equal(fl[ok], flr[ok])            # nonzero rule: |omega| decides


def test_additivity_over_loops():
    """Faces A (outer loops) and B (holes) queried separately and as one face."""
    wl = G.gen_c5(n_faces=400, grid=16, periodic_frac=0.0)
    faces = _faces_of(wl)
    multi = [i for i, (loops, _, _) in enumerate(faces) if len(loops) >= 2]
    assert len(multi) > 50
    sel = np.isin(wl["face_id"], multi)
    uv, fid = wl["uv"][sel], wl["face_id"][sel]
    remap = {f: k for k, f in enumerate(multi)}
    lid = np.array([remap[f] for f in fid], np.int32)
    wa, fa = _query(H.make_wl([(faces[f][0][:1], faces[f][1], faces[f][2]) for f in multi], uv, lid))
    wb, fb = _query(H.make_wl([(faces[f][0][1:], faces[f][1], faces[f][2]) for f in multi], uv, lid))
    wab, fab = _query(H.make_wl([faces[f] for f in multi], uv, lid))
    ok = (fa < 2) & (fb < 2) & (fab < 2)
    assert ok.mean() > 0.99
    assert np.array_equal(wab[ok], wa[ok] + wb[ok])   # integers: exact


@pytest.mark.parametrize("k", [3, -7])
def test_power_of_two_scaling_is_exact(k):
    s = 2.0 ** k
    wl = G.gen_c5(n_faces=300, grid=24)              # exact lattice data: periods on the 2^-40 grid scale exactly too
    w, fl = _query(wl)
    sc = dict(wl)
    sc["ctrl_uv"] = wl["ctrl_uv"] * s
    sc["uv"] = wl["uv"] * s
    sc["face_domain"] = wl["face_domain"] * s
    sc["eps"] = wl["eps"] * s
    w2, fl2 = _query(sc, eps=wl["eps"] * s)
    assert np.array_equal(fl, fl2)
    assert np.array_equal(np.nan_to_num(w, nan=9.0), np.nan_to_num(w2, nan=9.0))


def test_two_handles_on_two_streams():
    wl1 = G.gen_c5(n_faces=600, grid=32, seed=21)
    wl2 = G.gen_c2(n_queries=300_000, seed=22)
    ref1, ref2 = _query(wl1), _query(wl2)
    f1, f2 = wn.Faces.from_workload(wl1), wn.Faces.from_workload(wl2)
    dev = torch.device("cuda", 0)
    T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    q1 = (T(wl1["face_id"], torch.int32), T(wl1["uv"], torch.float64))
    q2 = (T(wl2["face_id"], torch.int32), T(wl2["uv"], torch.float64))
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    outs = []
    for _ in range(4):                                 # interleaved launches on both streams
        with torch.cuda.stream(s1):
            r1 = f1.query(*q1, stream=s1)
        with torch.cuda.stream(s2):
            r2 = f2.query(*q2, stream=s2)
        outs.append((r1, r2))
    torch.cuda.synchronize()
    for r1, r2 in outs:
        assert np.array_equal(r1.flag.cpu().numpy(), ref1[1]) and np.array_equal(r2.flag.cpu().numpy(), ref2[1])
        assert np.array_equal(np.nan_to_num(r1.winding.cpu().numpy(), nan=9.0), np.nan_to_num(ref1[0], nan=9.0))
        assert np.array_equal(np.nan_to_num(r2.winding.cpu().numpy(), nan=9.0), np.nan_to_num(ref2[0], nan=9.0))
    f1.close()
    f2.close()

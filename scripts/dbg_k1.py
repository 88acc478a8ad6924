import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_25159_b200 as wn
from tests import helpers as H
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "hodo_ref.py")).read())
P = np.array([[1., 0], [1, 1], [0, 1]]); w = np.array([1, math.sqrt(.5), 1])
P2 = np.array([[0, 0], [0.3, 0.9], [0.8, -0.4], [1, 0.2]]); w2 = np.array([1, 2, 0.5, 1.5])
segs = [(P, w), (P2, w2)]
wl = H.make_wl([([segs], 0, (0, 1, 0, 1))])
out = wn.segment_prep(wl["ctrl_uv"], wl["ctrl_w"], wl["seg_degree"]).cpu().numpy()
np.set_printoptions(precision=6, linewidth=200)
for (P_, w_), row in zip(segs, out):
    n = len(P_) - 1
    Hh = np.concatenate([w_[:, None] * P_, w_[:, None]], 1)
    print("gpu", row)
    print("ref B", min(floater(n, Hh), hodo(n, Hh)), "pieces", [min(floater(n, Hh), hodo(n, Hh), 8 * min(floater(n, pc), hodo(n, pc))) for pc in pieces(n, Hh)])

import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2510_25159_b200 as wn
from wn_workloads import configs as G
wl = G.gen_c5()
dev = torch.device("cuda", 0)
T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)
geo = [T(wl["ctrl_uv"], torch.float64), T(wl["ctrl_w"], torch.float64), T(wl["seg_degree"], torch.int32),
       T(wl["loop_seg_off"], torch.int32), T(wl["face_loop_off"], torch.int32), T(wl["face_periodic"], torch.uint8),
       T(wl["face_domain"], torch.float64)]
for i in range(6):
    if i == 5: os.environ["WN_TRACE"] = os.environ.get("TRACE_MODE", "1")
    wn.Faces.build(*geo).close()
    torch.cuda.synchronize()

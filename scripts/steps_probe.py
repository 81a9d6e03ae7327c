"""Per-step phase times of successive device-resident treecode calls (warm-up diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_12498_b200 as S
from bench import CONFIGS, make_inputs
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]
peak_first = len(sys.argv) > 2 and sys.argv[2] == "peak"
ps, tg = make_inputs(cfg)
n = cfg["n"]
dsrc = torch.from_numpy(np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal])).cuda()
dout = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"])
b = dsrc.data_ptr(); st = n * 24
if peak_first:
    print("peak", S.fp64_peak(0.3))
for i in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t = time.time()
    e0.record()
    r = S.treecode_velocity_device(b, b + st, b + 2 * st, b + 3 * st, n, prm, dout.data_ptr(),
                                   stream=torch.cuda.current_stream().cuda_stream)
    e1.record(); torch.cuda.synchronize()
    print(f"step {i}: events {e0.elapsed_time(e1):7.2f} ms wall {1e3*(time.time()-t):7.2f} total {1e3*r.time_total_s:7.2f} "
          f"build {1e3*r.time_build_s:6.2f} mom {1e3*r.time_moments_s:6.2f} far {1e3*r.time_far_s:6.2f} near {1e3*r.time_near_s:6.2f}", flush=True)

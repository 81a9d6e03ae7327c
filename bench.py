#!/usr/bin/env python
"""Benchmark of the treecode evaluation hot path (BASELINE.json metric).

One step = one full treecode evaluation (tree build -> moments -> far field ->
near field -> velocities in original order) of BASELINE.json configs[1]
(N = 1,000,000 uniform-cube particles, theta 0.5, p 8, N0 2000, Stokeslet +
stresslet, targets = sources) unless --config says otherwise.

value : target velocities/s, whole job, inputs resident in HBM, device time
        (CUDA events on the launching stream), max over ranks.
e2e   : the same metric through the public C ABI with pinned HOST buffers:
        H2D of the particle arrays, the treecode, D2H of the velocities.
accuracy : the other half of the BASELINE metric -- relative L2 error against the
        direct sum on the reference's strided 1,000-target subset (bench.hpp:235-256),
        the reference's own error on the same subset, and the distance to the
        reference treecode there.

--gpus N (N > 1) without torchrun re-launches itself under torch.distributed.run with
N ranks (NCCL; gloo when the box has fewer than N GPUs, ranks then share them).  Every
rank rebuilds the tree and moments (bit-identical) and evaluates its work-balanced shard
of the key-ordered target batches; the epilogue kernel stores each shard straight
into rank 0's output over NVLink (CUDA IPC), or --gather nccl all-gathers batch-order
slices.

--impl reference runs the reference's own CPU treecode (the headers under
/root/reference compiled in place, oracle/_ref/libstref.so) on all usable host cores,
with inputs from the oracle's generator: the product library is never loaded on that arm.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    "cfg0": dict(kind="cube", n=10_000, order=6, theta=0.5, n0=500, targets=None,
                 desc="cfg0: N=10,000 uniform cube [-0.5,0.5)^3, theta=0.5, p=6, N0=500"),
    "cfg1": dict(kind="cube", n=1_000_000, order=8, theta=0.5, n0=2000, targets=None,
                 desc="cfg1: N=1,000,000 uniform cube [-0.5,0.5)^3, theta=0.5, p=8, N0=2000"),
    "cfg2": dict(kind="sphere", n=4_000_000, order=10, theta=0.7, n0=2000, targets=None,
                 desc="cfg2: N=4,000,000 uniform on the unit sphere, nu = normal, theta=0.7, p=10, N0=2000"),
    "cfg3": dict(kind="cube", n=16_000_000, order=8, theta=0.5, n0=4000, targets=None,
                 desc="cfg3: N=16,000,000 uniform cube, theta=0.5, p=8, N0=4000"),
    "cfg4": dict(kind="mixture", n=8_000_000, order=8, theta=0.6, n0=2000, targets=8_000_000,
                 desc="cfg4: 8M sources from 16 Gaussians (sigma 0.05) / 8M uniform disjoint targets, "
                      "theta=0.6, p=8, N0=2000"),
}
SRC_SEED, TGT_SEED = 12345, 67890
METRIC = "target velocities/s"
F_NEAR = 48  # reference-algorithmic flops per direct pair, both kernels
ACC_SAMPLE = 1000  # BASELINE cfg1: error vs direct on a 1,000-target subset
HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


def E(n):
    return (n + 1) * (n + 2) * (n + 3) // 6


def f_far(p):
    """Reference-algorithmic flops per accepted particle-cluster pair, both kernels
    (Coulomb recurrence + Eq. 25 + Eq. 30 as the reference writes them)."""
    P = p + 2
    return (11 * E(P) + 5 * P - 16) + 41 * E(p) + (147 * E(p) + 3) + 6


def far_executed_flops(P):
    """FP64 flops the far kernels EXECUTE per accepted pair at harmonic order P (= p + 2 with
    stresslets): far_eval<P> in csrc/far_eval.cuh counted op by op (FMA = 2) plus the pair's
    geometry in the calling loop (dx and r^2 as the MAC computes them: 2 DMUL + 5 DADD as
    the compiler emits them).  tests/test_sass_counts.py checks this against the
    DFMA/DMUL/DADD count of the event loop in the built SASS of k_far_list<P> and k_feval<P>,
    tests/test_gpu_far_flops.py against ncu's executed counts on a B200."""
    fma = mul = add = 0
    mul += 2; fma += 3          # rsqrt_dp correction
    mul += 3                    # unit direction
    mul += 3                    # grade 0: three Phi columns
    for n in range(1, P + 1):
        if n >= 2:
            mul += 2 * n - 3; fma += 2 * n - 3   # w_n^m = z w_{n-1}^m + beta w_{n-2}^m, m <= n-2
            mul += 4; fma += 2                   # m = n-1, m = n
        mul += 1                                 # r^-(n+1)
        cols = 4 if n < P else 1                 # the top grade carries Psi only
        mul += cols; fma += cols * 2 * n         # contraction over the 2n+1 harmonics
        fma += cols                              # accumulate the grade
    fma += 3; add += 3                           # u_i += Phi_i + dx_i Psi
    add += 5; mul += 2                           # pair geometry in the event loop
    return 2 * fma + mul + add


def far_lds_per_pair(P):
    """Broadcast shared-memory loads of folded weights per accepted pair in k_far_list<P>
    (csrc/far_eval.cuh): (LDS.128, LDS.64).  Two LDS.128 per harmonic coefficient (four
    weight columns); the top grade's lone Psi column and grade 0's third Phi column as
    LDS.64.  (199, 22) at P = 10, matching the SASS."""
    return 1 + sum(2 * (2 * n + 1) for n in range(1, P)), 1 + (2 * P + 1)


def far_lds_clk_per_pair(P):
    """SM clocks per warp event the weight loads hold the shared-memory pipe: a broadcast
    LDS.128 costs 2, an LDS.64 1 (scripts/micro/lds_split.cu, profiles/r02_lds_split.md)."""
    l128, l64 = far_lds_per_pair(P)
    return LDS128_CLK * l128 + LDS64_CLK * l64


LDS128_CLK = 2.0  # SM clocks per warp-wide broadcast LDS.128 (profiles/r02_lds_split.md)
LDS64_CLK = 1.0   # ... per broadcast LDS.64


def moment_flops_per_incidence(p):
    """Reference-algorithmic flops per particle-cluster incidence of compute_moments
    (25 E(p) + 11, moments.hpp:34-80)."""
    return 25 * E(p) + 11


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "usable_cores": usable, "os_cpu_count": os.cpu_count()}


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        v = float(json.load(open(p))["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback of B200_PROFILING.md (MEASURED_PEAKS.json absent)"


class ClockSampler:
    """SM clocks + throttle reasons sampled in-process through NVML (pynvml) every 25 ms
    during the timed region (lighter than an nvidia-smi subprocess next to the step)."""

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.lines = []  # (wall time, sm MHz, max MHz, reasons bitmask)
        self.window = (0.0, float("inf"))
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.idx)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.N = None
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                mx = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.lines.append((time.time(), sm, mx, rs))
            except Exception:
                pass
            self._stop.wait(0.025)

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while self.t is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def mark(self, start, end):
        self.window = (start, end)

    def __exit__(self, *a):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=2)

    def summary(self):
        bits = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
                "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
        sm, mx, reasons = [], None, set()
        for ts, f, m, rs in self.lines:
            if not (self.window[0] - 0.1 <= ts <= self.window[1] + 0.1):
                continue
            sm.append(float(f))
            mx = float(m)
            for nm, b in bits.items():
                if rs & b:
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0, "source": "nvml"}
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(np.min(sm)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml (pynvml), 25 ms"}


def allgather_batch_slices(dist, ubatch, t0, t1, world):
    """All-gather every rank's contiguous batch-order slice [t0, t1) of `ubatch` (n, 3) into
    every rank's `ubatch` (one all-gather of the ranges, one all-gather of equal-length
    padded slices; works on NCCL and gloo)."""
    import torch
    dev = ubatch.device
    rng = torch.tensor([t0, t1], dtype=torch.int64, device=dev)
    ranges = [torch.empty_like(rng) for _ in range(world)]
    dist.all_gather(ranges, rng)
    ranges = [tuple(int(v) for v in r.tolist()) for r in ranges]
    maxlen = max(1, max(b - a for a, b in ranges))
    send = torch.zeros((maxlen, 3), dtype=ubatch.dtype, device=dev)
    send[: t1 - t0] = ubatch[t0:t1]
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send)
    for (a, b), piece in zip(ranges, recv):
        ubatch[a:b] = piece[: b - a]
    return ranges


def make_inputs(cfg):
    """GPU arm: the product's host generator (st_generate)."""
    import paper_1811_12498_b200 as S
    ps = S.generate(cfg["kind"], cfg["n"], SRC_SEED, True)
    tg = S.generate("points", cfg["targets"], TGT_SEED).position if cfg["targets"] else None
    return ps, tg


def make_reference_inputs(cfg):
    """Reference arm and CPU checks: the oracle's own C generator (or_generate), so the
    reference arm never loads the product library.  Same bytes as make_inputs (pinned by
    SHA-256 in tests/test_inputs_io.py)."""
    from oracle import oracle as O
    ps = O.generate(cfg["kind"], cfg["n"], SRC_SEED, True)
    tg = O.generate("points", cfg["targets"], TGT_SEED)["position"] if cfg["targets"] else None
    return ps, tg


def accuracy_subset(nt):
    """The reference harness's strided direct sample, i * floor(n / sample) (bench.hpp:235-241)."""
    if nt <= ACC_SAMPLE:
        return np.arange(nt, dtype=np.int64)
    stride = nt // ACC_SAMPLE
    return np.arange(ACC_SAMPLE, dtype=np.int64) * stride


# ----------------------------------------------------------------------------- CPU reference
def cpu_reference_sample(ps, tg, cfg, threads, sample, ctx=None):
    """Reference CPU treecode (oracle/_ref) on a bounded sample: build + moments in full,
    traversal of `sample` strided targets on `threads` threads, extrapolated to all N
    targets (the reference's own --direct-sample idiom, bench.hpp:247-248)."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    own = ctx is None
    if own:
        ctx = O.RefContext(ps, cfg["order"], cfg["theta"], cfg["n0"], True, True, True, workers=threads)
    t1 = time.perf_counter()
    nt = cfg["targets"] or cfg["n"]
    stride = max(1, nt // sample)
    idx = np.arange(0, nt, stride)[:sample]
    t2 = time.perf_counter()
    if tg is None:
        ctx.eval(src_idx=idx, threads=threads)
    else:
        ctx.eval(xyz=tg[idx], threads=threads)
    t3 = time.perf_counter()
    tb = (t1 - t0) if own else (ctx.t_build + ctx.t_moments)
    full = tb + (t3 - t2) * nt / len(idx)
    return nt / full, dict(build_moments_s=tb, sample_targets=len(idx), sample_traverse_s=t3 - t2), ctx


def reference_accuracy(ps, tg, cfg, threads, ctx, u_tree_subset=None):
    """The reference's own error vs direct on the strided subset, plus its treecode there."""
    from oracle import oracle as O
    nt = cfg["targets"] or cfg["n"]
    idx = accuracy_subset(nt)
    if u_tree_subset is None:
        u_tree_subset = ctx.eval(src_idx=idx, threads=threads)[0] if tg is None else \
            ctx.eval(xyz=tg[idx], threads=threads)[0]
    if tg is None:
        u_dir = O.ref_direct_at(ps, idx, threads=threads)
        how = "reference contracted_direct_velocity_at (oracle/_ref)"
    else:  # the reference has no direct sum at disjoint points: the C restatement's (bit-pinned)
        u_dir = O.or_direct_points(ps, tg[idx], threads=threads)
        how = "oracle C restatement or_direct_points (the reference has no disjoint-target direct sum)"
    return idx, u_tree_subset, u_dir, how


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libstref.so not built"}))
        return
    hi = host_info()
    threads = hi["usable_cores"]
    ps, tg = make_reference_inputs(cfg)
    nt = cfg["targets"] or cfg["n"]
    full_ok = tg is None and cfg["n"] <= args.ref_full_max
    # warm-up: bounded samples (page in the code and the inputs)
    for _ in range(min(args.warmup, 1)):
        _, _, c = cpu_reference_sample(ps, tg, cfg, threads, 256)
        c.close()
    detail = {}
    if full_ok:
        # the whole workload once, as the reference's public parallel_velocity runs it
        # (engine.hpp:194-196) with workers = every usable core; BASELINE.md section 3
        t0 = time.perf_counter()
        u, stats, times = O.ref_parallel_velocity(ps, cfg["order"], cfg["theta"], cfg["n0"], True, True, True,
                                                  workers=threads)
        wall = time.perf_counter() - t0
        value = nt / wall
        steps = 1
        idx = accuracy_subset(nt)
        ctx = O.RefContext(ps, cfg["order"], cfg["theta"], cfg["n0"], True, True, True, workers=threads)
        v_x, info_x, _ = cpu_reference_sample(ps, tg, cfg, threads, args.ref_sample, ctx=ctx)
        _, u_sub, u_dir, how = reference_accuracy(ps, tg, cfg, threads, ctx, u_tree_subset=u[idx])
        ctx.close()
        mode = (f"full run: parallel_velocity on all {nt} targets, {threads} workers "
                f"(wall {wall:.1f} s: build {times['build']:.2f} s, moments {times['moments']:.2f} s, "
                f"traverse {times['traverse']:.1f} s)")
        detail = {"wall_s": wall, "phase_s": times, "stats": stats,
                  "extrapolated_cross_check": {"value": v_x, **info_x,
                                               "note": "strided-sample extrapolation (bench.hpp:247-248)"}}
    else:
        vals = []
        ctx = None
        for _ in range(args.steps):
            if ctx is not None:
                ctx.close()
            v, info, ctx = cpu_reference_sample(ps, tg, cfg, threads, args.ref_sample)
            vals.append(v)
        value = float(np.mean(vals))
        steps = args.steps
        _, u_sub, u_dir, how = reference_accuracy(ps, tg, cfg, threads, ctx)
        ctx.close()
        mode = (f"sampled: full build + moments, traversal of {info['sample_targets']} strided targets on "
                f"{threads} threads, extrapolated to {nt} (bench.hpp:247-248; a full run would take "
                f"~{nt / value / 60:.0f} min)")
        detail = {"samples": info, "per_step_values": vals}
    err = O.relative_error(u_dir, u_sub)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "targets/s", "n_gpus": world,
        "steps": steps, "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": nt / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64, oracle/or_generate)",
        "config": config_block(cfg, args, world=1),
        "cpu_baseline": {"value": value, "unit": "targets/s", "cores": threads, "kind": "reference",
                         "sample": mode, **hi},
        "e2e": {"value": value, "unit": "targets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "accuracy": {"E_vs_direct": err, "subset": f"{len(u_sub)} strided targets (bench.hpp:235-241)",
                     "direct": how},
        "detail": detail,
    }
    print(json.dumps(line), flush=True)


def config_block(cfg, args, world):
    par = "one GPU"
    if world > 1:
        split = args.gather == "peer" and args.moments == "split"
        par = (f"targets sharded over {world} GPUs by work-balanced key-ordered batches, tree replicated, "
               + ("moment pass split by subtrees with the weight rows exchanged over NCCL" if split
                  else "moments replicated")
               + (", shards stored into rank 0's output by the epilogue kernel (CUDA IPC, NVLink)"
                  if args.gather == "peer" else ", batch-order slices all-gathered over NCCL"))
    return {"workload": cfg["desc"], "n_sources": cfg["n"], "n_targets": cfg["targets"] or cfg["n"],
            "order": cfg["order"], "theta": cfg["theta"], "leaf_capacity": cfg["n0"], "shrink": True,
            "kernels": "stokeslet+stresslet", "seeds": [SRC_SEED, TGT_SEED] if cfg["targets"] else [SRC_SEED],
            "l2": "flushed between timed steps (512 MiB write, outside the step events)",
            "parallelism": par}


# ----------------------------------------------------------------------------- GPU arm
def relaunch_command(args_list, n, port):
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(args_list)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args):
    """`bench.py --gpus N` with N > 1 and no torchrun environment: run N ranks under
    torch.distributed.run.  NCCL when the box has N GPUs; otherwise gloo with the ranks
    sharing the GPUs (a plumbing check, labelled as such in the line)."""
    env = dict(os.environ)
    ngpu = 0
    try:
        import torch
        ngpu = torch.cuda.device_count()
    except Exception:
        pass
    if ngpu < args.gpus:
        env["ST_BENCH_BACKEND"] = "gloo"
        print(f"[bench] {ngpu} GPU(s) visible for --gpus {args.gpus}: gloo, ranks share GPUs "
              "(plumbing check, not a scaling measurement)", file=sys.stderr, flush=True)
    cmd = relaunch_command(sys.argv[1:], args.gpus, free_port())
    return subprocess.run(cmd, env=env).returncode


def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1811_12498_b200 as S

    world, rank, local = dist_env()
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    ngpu = torch.cuda.device_count()
    local = local % max(1, ngpu)
    torch.cuda.set_device(local)
    backend = None
    if world > 1:
        # NCCL on the driver's runs; ST_BENCH_BACKEND=gloo lets a one-GPU box run the N>1
        # path (ranks then share the GPU; their kernels never wait on each other)
        backend = os.environ.get("ST_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    # inputs: generated on rank 0 host, broadcast over NCCL (replicated sources)
    nt = cfg["targets"] or cfg["n"]
    n = cfg["n"]
    if rank == 0:
        ps, tg = make_inputs(cfg)
        host = np.concatenate([ps.position, ps.force_weight, ps.dipole_weight, ps.normal], axis=0)
    else:
        ps, tg, host = None, None, None
    dsrc = torch.empty((4 * n, 3), dtype=torch.float64, device=dev)
    dtg = torch.empty((nt, 3), dtype=torch.float64, device=dev) if cfg["targets"] else None
    if rank == 0:
        dsrc.copy_(torch.from_numpy(host))
        if dtg is not None:
            dtg.copy_(torch.from_numpy(tg))
    if world > 1:
        dist.broadcast(dsrc, 0)
        if dtg is not None:
            dist.broadcast(dtg, 0)
    dout = torch.zeros((nt, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    prm = S.TreecodeParams(order=cfg["order"], theta=cfg["theta"], leaf_capacity=cfg["n0"], shrink=True)
    base = dsrc.data_ptr()
    stride = n * 3 * 8
    ptrs = (base, base + stride, base + 2 * stride, base + 3 * stride)

    peer_out = None
    if world > 1 and args.gather == "peer":
        # fused gather: rank 0 exports its output buffer (CUDA IPC); every rank's epilogue
        # kernel stores its shard's velocities straight into it, in original order, over
        # NVLink; a one-element all-reduce after the call orders the ranks
        obj = [S.ipc_export(dout.data_ptr()) if rank == 0 else None]
        dist.broadcast_object_list(obj, 0)
        peer_out = dout.data_ptr() if rank == 0 else S.ipc_open(*obj[0])
        done = torch.zeros(1, dtype=torch.float32, device=dev)
        from paper_1811_12498_b200.distributed import collective_exchange
        exchange = collective_exchange(dist, local)
    elif world > 1:
        dbatch = torch.zeros((nt, 3), dtype=torch.float64, device=dev)
        torig = torch.empty(nt, dtype=torch.int32, device=dev)

    def step():
        tp = None if dtg is None else dtg.data_ptr()
        ntp = nt if dtg is not None else 0
        if world == 1:
            return S.treecode_velocity_device(*ptrs, n, prm, dout.data_ptr(), targets_ptr=tp, n_targets=ntp,
                                              stream=sptr)
        if peer_out is not None:
            if args.moments == "split":
                # each rank computes its subtrees' moments; the weight rows are exchanged by
                # one broadcast per rank on the call's stream (NCCL over NVLink)
                r = S.treecode_velocity_device_split(*ptrs, n, prm, peer_out, exchange, targets_ptr=tp, n_targets=ntp,
                                                     shard=rank, n_shards=world, stream=sptr)
            else:
                r = S.treecode_velocity_device(*ptrs, n, prm, peer_out, targets_ptr=tp, n_targets=ntp, shard=rank,
                                               n_shards=world, stream=sptr)
            dist.all_reduce(done)  # every shard's stores into rank 0's buffer have completed
            return r
        # every rank: same tree/moments, its work-balanced slice of the key-ordered batches in
        # batch order; NCCL all-gather of the slices over NVLink; scatter to original order
        t0, t1, r = S.treecode_shard_device(*ptrs, n, prm, dbatch.data_ptr(), torig.data_ptr(), targets_ptr=tp,
                                            n_targets=ntp, shard=rank, n_shards=world, stream=sptr)
        allgather_batch_slices(dist, dbatch, t0, t1, world)
        S.unbatch_device(nt, torig.data_ptr(), dbatch.data_ptr(), dout.data_ptr(), stream=sptr)
        return r

    peak = S.fp64_peak(0.3)
    clocks = ClockSampler(local).__enter__()
    clocks.wait_first()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    near_t = far_t = 0.0
    stats = None
    launches = 0
    phases = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = time.time()
    for k in range(args.steps):
        flush.fill_(float(k))
        ev[k][0].record(stream)
        r = step()
        ev[k][1].record(stream)
        near_t += r.time_near_s
        far_t += r.time_far_s
        launches += r.gpu_launches
        stats = r.stats
        phases.append([round(1e3 * x, 2) for x in (r.time_build_s, r.time_moments_s, r.time_far_s, r.time_near_s,
                                                   r.time_total_s)])
    torch.cuda.synchronize()
    clocks.mark(t_start, time.time())
    if world > 1:
        dist.barrier()
    clocks.__exit__()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    my_ms = float(sum(step_ms))
    t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms = t.item()
    value = nt * args.steps / (tot_ms * 1e-3)
    u_final = dout[accuracy_subset(nt)].cpu().numpy() if rank == 0 else None  # the timed steps' output

    # ---- e2e through the public C ABI with pinned host buffers (H2D + treecode + D2H)
    hsrc = torch.empty((4 * n, 3), dtype=torch.float64).pin_memory()
    hout = torch.empty((nt, 3), dtype=torch.float64).pin_memory()
    htg = torch.empty((nt, 3), dtype=torch.float64).pin_memory() if dtg is not None else None
    if rank == 0:
        hsrc.copy_(torch.from_numpy(host))
        if htg is not None:
            htg.copy_(torch.from_numpy(tg))
    h2d_bytes = hsrc.numel() * 8 + (htg.numel() * 8 if htg is not None else 0)
    d2h_bytes = hout.numel() * 8

    side = torch.cuda.Stream() if world == 1 else None
    w_ready = torch.cuda.Event() if world == 1 else None
    t_ready = torch.cuda.Event() if world == 1 else None
    w_start = torch.cuda.Event() if world == 1 else None

    def e2e_step():
        if world == 1:
            # positions (and targets) on the compute stream; the weight arrays on a side
            # stream, overlapping the tree build (st_treecode_velocity_device_ev waits for
            # them after the build, the way st_treecode_velocity_ex does for host arrays)
            dsrc[:n].copy_(hsrc[:n], non_blocking=True)
            # disjoint targets, then the weights, start once the positions are in (the
            # previous step is done with dsrc and dtg too): sharing the PCIe link with the
            # positions would only delay the build; the targets' ordering runs beside it
            w_start.record(stream)
            side.wait_event(w_start)
            with torch.cuda.stream(side):
                if dtg is not None:
                    dtg.copy_(htg, non_blocking=True)
                    t_ready.record(side)
                dsrc[n:].copy_(hsrc[n:], non_blocking=True)
                w_ready.record(side)
            tp = None if dtg is None else dtg.data_ptr()
            S.treecode_velocity_device(*ptrs, n, prm, dout.data_ptr(), targets_ptr=tp,
                                       n_targets=nt if dtg is not None else 0, stream=sptr,
                                       weights_event=w_ready.cuda_event,
                                       targets_event=t_ready.cuda_event if dtg is not None else 0)
            hout.copy_(dout, non_blocking=True)
            return
        if rank == 0:
            dsrc.copy_(hsrc, non_blocking=True)
            if dtg is not None:
                dtg.copy_(htg, non_blocking=True)
        dist.broadcast(dsrc, 0)
        if dtg is not None:
            dist.broadcast(dtg, 0)
        step()
        if rank == 0:
            hout.copy_(dout, non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    for k in range(args.steps):
        flush.fill_(float(k))
        ee[k][0].record(stream)
        e2e_step()
        ee[k][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ee)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_val = nt * args.steps / (e2e_ms.item() * 1e-3)
    if rank == 0:
        u_e2e = hout.numpy().copy()
        assert np.isfinite(u_e2e).all()
    e2e = {"value": e2e_val, "unit": "targets/s", "h2d_bytes_per_step": int(h2d_bytes) if rank == 0 else 0,
           "d2h_bytes_per_step": int(d2h_bytes),
           "path": "st_treecode_velocity_device_ev2 with per-step H2D of pinned particle arrays (positions "
                   "first; disjoint targets, then the weights, on a side stream overlapping the tree build) and "
                   "D2H of the velocities "
                   "(CUDA events, max over ranks)",
           "step_ms": [round(a.elapsed_time(b), 3) for a, b in ee]}
    if world == 1:
        # the reference-facing host call itself (st_treecode_velocity, engine.hpp:194-196) on
        # pinned host arrays: wall clock around the synchronous call, median of the timed steps
        hp = hsrc.numpy()
        pps = S.ParticleSet(hp[:n], hp[n:2 * n], hp[2 * n:3 * n], hp[3 * n:])
        htgt = htg.numpy() if htg is not None else None

        def host_call(p, tt):
            walls = []
            for k in range(args.steps + 1):
                t0 = time.perf_counter()
                res = S.treecode_velocity_targets(p, tt, prm)
                walls.append(time.perf_counter() - t0)
            assert np.isfinite(res.velocity).all()
            return float(np.median(walls[1:]))

        w = host_call(pps, htgt)
        e2e["host_api"] = {"value": nt / w, "unit": "targets/s", "wall_ms_median": 1e3 * w,
                           "call": "paper_1811_12498_b200.treecode_velocity -> st_treecode_velocity_ex, "
                                   "pinned host arrays",
                           "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(d2h_bytes)}
        w = host_call(ps, tg)
        e2e["host_api_pageable"] = {"value": nt / w, "unit": "targets/s", "wall_ms_median": 1e3 * w,
                                    "call": "same call, pageable host arrays (numpy)",
                                    "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(d2h_bytes)}

    # ---- this rank's roofline: near field (dominant), far field, moment pass
    P = cfg["order"] + 2
    near_s = near_t / args.steps
    far_s = far_t / args.steps
    near_flops = F_NEAR * stats.direct_pairs
    far_exec = far_executed_flops(P) * stats.farfield_evals
    far_refeq = f_far(cfg["order"]) * stats.farfield_evals
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.config, {}).get("near_dram_bytes_per_launch")
        except Exception:
            traffic = None
    ach_near = near_flops / near_s * 1e-12 if near_s > 0 else None
    ach_far = far_exec / far_s * 1e-12 if far_s > 0 else None
    moments = measure_moments(S, step, cfg, ps if rank == 0 else None, peak, world) if world == 1 else None
    roof = {"bound": "fp64",
            "kernel": "k_neval (near-field leaf direct sums; CUDA events around its launches)",
            "achieved": ach_near, "peak": peak, "unit": "TFLOP/s",
            "frac": (ach_near / peak) if ach_near else None,
            "traffic": traffic if world == 1 else None,
            "flops_per_launch": near_flops, "flop_convention": "48 flop per direct pair (reference count; the "
                                                               "kernel executes 30 DP ops + 1 MUFU.RSQ64H per pair)",
            "peak_source": "live DFMA-loop probe in this run (MEASURED_PEAKS.json has no FP64 figure)",
            "far": {"kernel": "k_far_list (dense far events) + k_feval (sparse far events, packed)",
                    "achieved": ach_far, "frac": (ach_far / peak) if ach_far else None,
                    "flops_per_launch": far_exec,
                    "flop_convention": f"executed: {far_executed_flops(P)} FP64 flop per accepted pair at "
                                       f"harmonic order P={P} (far_eval<P> op count, checked against the "
                                       "SASS by tests/test_sass_counts.py)",
                    "reference_equivalent": {
                        "flops_per_launch": far_refeq, "flop_per_pair": f_far(cfg["order"]),
                        "tflops": far_refeq / far_s * 1e-12 if far_s > 0 else None,
                        "note": "the reference's Cartesian contraction would need "
                                f"{f_far(cfg['order']) / far_executed_flops(P):.1f}x these flops for "
                                "the same pairs; not a roofline fraction"}},
            "moments": moments,
            "near_s": near_s, "far_s": far_s}
    # the far field's other ceiling: every weight reaches the lanes as a broadcast
    # shared-memory load, 2 SM clocks per warp-wide LDS.128 and 1 per LDS.64 whatever the
    # lanes' addresses -- above the DP pipe's 0.5 clock per DFMA at this instruction mix, so
    # the shared-memory pipe binds first
    sm_clk_hz = 1e6 * (clocks.summary().get("sm_mhz") or 0.0)
    if far_s > 0 and sm_clk_hz > 0:
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        l128, l64 = far_lds_per_pair(P)
        clk = far_lds_clk_per_pair(P)
        ceiling = sms * sm_clk_hz * 32.0 / clk
        achieved = stats.farfield_evals / far_s
        roof["far"]["lds_bound"] = {
            "lds128_per_pair": l128, "lds64_per_pair": l64, "clk_per_warp_event": clk,
            "clk_per_warp_lds128": LDS128_CLK, "clk_per_warp_lds64": LDS64_CLK, "sms": sms, "sm_hz": sm_clk_hz,
            "ceiling_pairs_per_s": ceiling, "achieved_pairs_per_s": achieved, "frac": achieved / ceiling,
            "note": "pairs of both far kernels (k_feval's sparse events read weights from global memory) "
                    "against the dense kernel's shared-memory ceiling at full lanes"}
    mine = {"rank": rank, "ms_per_step": my_ms / args.steps, "near_s": near_s, "far_s": far_s,
            "near_frac": roof["frac"], "far_frac": roof["far"]["frac"],
            "direct_pairs": stats.direct_pairs, "farfield_evals": stats.farfield_evals}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)

    accuracy = None
    cpu = None
    if rank == 0:
        accuracy, cpu = accuracy_and_cpu(S, args, cfg, ps, tg, u_final, world)

    if rank == 0:
        slow = max(per_rank, key=lambda d: d["ms_per_step"])
        line = {
            "metric": METRIC, "value": value, "unit": "targets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
            "config": config_block(cfg, args, world), "e2e": e2e, "gpu_launches": launches,
            "roofline": roof if world == 1 else dict(roof, note=f"rank 0's kernels; slowest rank {slow['rank']}"),
            "accuracy": accuracy, "cpu_baseline": cpu, "clocks": clocks.summary(),
            "stats": {"farfield_evals": stats.farfield_evals, "direct_pairs": stats.direct_pairs,
                      "clusters_visited": stats.clusters_visited},
            "step_ms": step_ms,
            "step_phases_ms": {"columns": ["build", "moments", "far", "near", "treecode_total"], "steps": phases},
        }
        if world > 1:
            line["backend"] = backend + ("" if backend == "nccl" else
                                         f" ({ngpu} GPU(s) shared by {world} ranks: plumbing check, "
                                         "not a scaling measurement)")
            line["per_rank"] = per_rank
            line["slowest_rank"] = slow
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        if peer_out is not None and rank != 0:
            S.ipc_close(peer_out)
        dist.destroy_process_group()


def measure_moments(S, step, cfg, ps, peak, world):
    """Moment pass (K2: leaf moments + M2M + fold) alone: the same call with
    ST_MOMENTS_INLINE=1, so nothing overlaps it and time_moments_s is its duration.
    Algorithmic bytes: the 96-B source records read once + the folded weights written once;
    FP64: reference-algorithmic 25 E(p) + 11 flop per particle-cluster incidence over all
    clusters (what compute_moments executes, moments.hpp:34-80), and the same per particle
    at the leaves only (what this pass computes from particles; M2M shifts the rest)."""
    import torch
    os.environ["ST_MOMENTS_INLINE"] = "1"
    try:
        ts = []
        for _ in range(4):
            r = step()
            ts.append(r.time_moments_s)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("ST_MOMENTS_INLINE", None)
    t = float(np.median(ts[1:]))
    n = cfg["n"]
    p = cfg["order"]
    P = p + 2
    incid = None
    ncl = None
    if ps is not None:
        T = S.build_tree(ps, cfg["n0"], True)
        ncl = int(T.ncl)
        incid = int(np.sum(T.end.astype(np.int64) - T.begin.astype(np.int64)))
    bytes_alg = 96 * n + (ncl or 0) * (P + 1) ** 2 * 4 * 8
    hbm, hbm_src = measured_hbm_peak()
    out = {"kernels": "k_moments (leaves, TMA tiles) + k_m2m (per level) + k_fold", "time_s": t,
           "algorithmic_bytes": bytes_alg, "achieved_gbs": bytes_alg / t * 1e-9, "hbm_peak_gbs": hbm,
           "hbm_frac": bytes_alg / t * 1e-9 / hbm, "hbm_peak_source": hbm_src,
           "timing": "ST_MOMENTS_INLINE=1 (moment pass serialised), median of 3 calls"}
    if incid is not None:
        f_ref = moment_flops_per_incidence(p) * incid
        f_leaf = moment_flops_per_incidence(p) * n
        out.update({"clusters": ncl, "particle_cluster_incidences": incid,
                    "reference_equivalent_tflops": f_ref / t * 1e-12,
                    "reference_equivalent_frac": f_ref / t * 1e-12 / peak,
                    "leaf_algorithmic_tflops": f_leaf / t * 1e-12,
                    "leaf_algorithmic_frac": f_leaf / t * 1e-12 / peak,
                    "bound": "max(bytes / HBM, flops / FP64): FP64 (>= 40 flop/B, SURVEY.md 8d)",
                    "binding_resource": "k_moments (leaf sums, most of the pass): the shared-memory pipe, 82% of "
                                        "its wavefront capacity at cfg4 (ncu: six broadcast LDS.128 of weights and "
                                        "six per-lane power loads per particle and warp for 24 FMAs per thread); "
                                        "k_fold: issue-bound on index arithmetic (FP64 7%); top M2M levels: "
                                        "latency-bound, ~73 us each (profiles/r02_moments_ncu.md, DESIGN.md sec. 9)"})
    return out


def accuracy_and_cpu(S, args, cfg, ps, tg, u_gpu_subset, world):
    """Rank 0: the accuracy block (GPU E vs direct, the reference's E on the same subset,
    rel L2 to the reference treecode there) and the bounded CPU baseline sample."""
    nt = cfg["targets"] or cfg["n"]
    idx = accuracy_subset(nt)
    sel = S.KernelSelection.both()
    if tg is None:
        u_dir = S.contracted_direct_velocity_at(ps, sel, idx)
        dir_how = "st_direct_velocity_at (GPU O(N^2) kernel k_direct)"
    else:  # direct sum at disjoint points: the treecode with theta -> 0 accepts no cluster
        u_dir = S.treecode_velocity_targets(ps, tg[idx], S.TreecodeParams(order=0, theta=1e-9,
                                                                          leaf_capacity=cfg["n0"])).velocity
        dir_how = "st_treecode_velocity_ex with theta=1e-9 (no far field: the direct sum, GPU)"
    acc = {"E_vs_direct": S.relative_error(u_dir, u_gpu_subset),
           "subset": f"{len(idx)} strided targets i*floor(N/{ACC_SAMPLE}) (bench.hpp:235-241)",
           "direct": dir_how}
    cpu = None
    if args.no_cpu_baseline or world > 1:
        return acc, cpu
    try:
        from oracle import oracle as O
        if not O.have_ref():
            return acc, {"value": None, "error": "oracle/_ref not built"}
        hi = host_info()
        threads = hi["usable_cores"]
        rps, rtg = make_reference_inputs(cfg)
        v, info, ctx = cpu_reference_sample(rps, rtg, cfg, threads, args.ref_sample)
        _, u_ref, u_ref_dir, how = reference_accuracy(rps, rtg, cfg, threads, ctx)
        ctx.close()
        e_ref = O.relative_error(u_ref_dir, u_ref)
        acc.update({"E_reference": e_ref, "E_rel_diff": abs(acc["E_vs_direct"] - e_ref) / e_ref,
                    "E_within_1pct": abs(acc["E_vs_direct"] - e_ref) <= 0.01 * e_ref,
                    "rel_l2_vs_reference_sample": O.relative_error(u_ref, u_gpu_subset),
                    "reference": "oracle/_ref (the reference compiled in place): treecode at the subset via "
                                 "detail::accumulate_velocity; direct: " + how})
        cpu = {"value": v, "unit": "targets/s", "cores": threads, "kind": "reference",
               "sample": f"reference treecode compiled in place, full build+moments, "
                         f"{info['sample_targets']} strided targets traversed on {threads} threads, "
                         f"extrapolated to {nt} targets ({info})", **hi}
    except Exception as e:  # reported, not fatal
        cpu = {"value": None, "error": str(e)}
    return acc, cpu


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPU count (default: WORLD_SIZE, else 1); N > 1 without torchrun re-launches under "
                         "torch.distributed.run")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg1", choices=sorted(CONFIGS))
    ap.add_argument("--ref-sample", type=int, default=4000)
    ap.add_argument("--ref-full-max", type=int, default=1_000_000,
                    help="reference arm: run the whole workload when N <= this (cfg0, cfg1), else sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--moments", default="split", choices=["split", "replicated"],
                    help="N>1: each rank computes its share of the moment pass and the ranks exchange the weight "
                         "rows (split), or every rank computes all of it (replicated)")
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N>1: shards stored into rank 0's buffer by the epilogue kernel over CUDA IPC "
                         "(peer), or batch-order slices all-gathered over NCCL and scattered (nccl)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return 0
    if args.gpus is not None and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    run_gpu(args, cfg)
    return 0


if __name__ == "__main__":
    sys.exit(main())

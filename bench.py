"""Benchmark: hypergradients/sec of the recycled hypergradient solve (BASELINE.json metric).

A "step" is one upper-level system of the replay protocol (experiments.py:390-463)
for every sample a rank owns: next_recycle (RGen-L(R): candidate basis, H W, J W,
projected GSVD, prepare_recycle) + the batched recycled-MINRES solve with the NSC
stop rule + J w, and the sample-ordered sum of the per-sample hypergradients
(all-gathered across ranks for N > 1).

Workload (default, N = 1): BASELINE configs[2] ("C3", the largest config that fits
one GPU): 64 samples of 256x256, 15x15 blur sigma 2.5, 2% noise, J = 8 learned 5x5
filters (p = 208), phi_eps with eps = 1e-2, recycle dimension 30, at most 300
Krylov iterations, NSC tolerance 1e-6.  `--config C2` runs configs[1].
Inputs: seeded synthetic data (problems.py); the frozen sequence of systems is
synthetic (theta drifting, xhat = x_true + slowly drifting smooth field).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run (one process per GPU, NCCL).  C3 is strong scaling: its fixed
64-sample batch is sharded across the ranks (distributed.shard); C2 / C4 are weak
scaling (8 / 16 samples per GPU, BASELINE's per-GPU share); C1 / C5 are
single-sample configs and run one replica per GPU.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

# load every CUDA module at context creation: a library kernel first used inside
# the timed region must not pay module loading there
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

STRATEGY = "RGen-L(R)-NSC"
DELTA = 1e-6
METRIC = "hypergradients/sec (recycled solve incl. HVP) + achieved HBM GB/s vs peak"
# how each config's samples map onto ranks (BASELINE.json configs): C3 shards one fixed
# 64-sample batch over 1/2/4/8 GPUs; C4 is 128 samples over 8 GPUs = 16 per GPU
SHARDING = {"C1": "replica", "C2": "weak", "C3": "strong", "C4": "weak", "C5": "replica"}
PER_GPU = {"C4": 16}
THREAD_ENV = ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--strategy", default=STRATEGY)
    ap.add_argument("--delta", type=float, default=DELTA)
    ap.add_argument("--sequence", default="solved",
                    help="solved (lower-level minimisers along the synthetic theta path, cached under .seqcache/), "
                         "recorded (device-recorded bilevel run), synthetic, or a krecycle-sequence-v1 directory")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=40.0, help="seconds of timed CPU work (cpu_baseline)")
    ap.add_argument("--ref-budget", type=float, default=150.0, help="seconds of timed CPU work (--impl reference)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def relaunch_if_needed(args):
    """`--gpus N` (N > 1) outside torchrun: run this script under torch.distributed.run."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def samples_for(name: str, cfg, world: int, rank: int):
    """(first global sample, count on this rank, total samples of the job)."""
    mode = SHARDING.get(name, "weak")
    if mode == "strong":
        from paper_2412_08264_b200.distributed import shard

        r = shard(cfg.batch, world, rank)
        return r.start, len(r), cfg.batch
    per = PER_GPU.get(name, cfg.batch)
    return rank * per, per, per * world


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region through NVML
    (in-process: no nvidia-smi fork of this large multi-threaded process, which
    stalled the host threads that drive the GPU); nvidia-smi only if NVML is absent."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nv = self._h = None
        try:  # import and initialise before the timed region, not inside it
            import pynvml as nv

            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(index)
            self._nv = nv
        except Exception:
            self._nv = None

    def _sample_nvml(self, nv, h):
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        flags = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        return [str(sm), str(mx)] + ["Active" if r & f else "Not Active" for f in flags]

    def _run(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                if nv is not None:
                    self.rows.append(self._sample_nvml(nv, h))
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                    parts = [p.strip() for p in out.stdout.strip().split(",")]
                    if len(parts) == 6:
                        self.rows.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def measured_fp64_peak():
    """fp64 DMMA peak measured on this pool's B200s (scripts/fp64_peak.cu, profiles/r2_fp64_peak.json)."""
    p = ROOT / "profiles" / "r2_fp64_peak.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["dmma_tflops"]), "measured (profiles/r2_fp64_peak.json dmma_tflops)"
    return 37.0, "fallback (nominal B200 fp64)"


def measured_traffic(config: str, kernel: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/traffic.json), or None when this config/kernel was not captured."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(config)
    if not d or d.get("kernel") != kernel:
        return None
    return int(d["dram_bytes_per_launch"]), d.get("source"), d.get("iterations_per_launch")


def krylov_bytes_per_iter(kernel, n, s, nsc, w):
    """Algorithmic HBM bytes per iteration per sample.
    RMINRES: 8n(21 + 3s + s_nsc) + the HVP's 8n(2 + w).
    Recycled CG: direction p = r + beta p - U mu (read r, p_old, U; write p), the
    stencil re-forming p on its tiles (r, p_old, U again), hp, the x/r update (read
    p, hp, x, r; write x, r) and the C^T r / Z^T r dots: 8n(12 + 3s + s_nsc) + 8n w.
    w = per-pixel weight vectors of the HVP (J filters, 3 for TV)."""
    if kernel == "kr_cg":
        return 8 * n * (12 + 3 * s + nsc) + 8 * n * w
    return 8 * n * (21 + 3 * s + nsc) + 8 * n * (2 + w)


def hvp_flops_per_pixel(cfg):
    """F = 8b + J(4q^2 + 2) + 2 (TV: 8b + 16)."""
    if cfg.reg == "tv":
        return 8 * cfg.blur_size + 16
    return 8 * cfg.blur_size + cfg.num_filters * (4 * cfg.kernel_size ** 2 + 2) + 2


def workload_text(name, cfg, count, total, args):
    return (f"{name}: {total} samples x {cfg.size}^2 ({count} on this rank), blur {cfg.blur_size} sigma "
            f"{cfg.blur_sigma}, J={cfg.num_filters} q={cfg.kernel_size}, s={cfg.recycle_dim}, max {cfg.max_iter} it, "
            f"{args.strategy} delta={args.delta}, {'recycled CG' if cfg.method == 'cg' else 'RMINRES'}")


# ---------------------------------------------------------------------------


# ---------------------------------------------------------------------------
# The workload's frozen sequence (the replay protocol's input, experiments.py:390-463).
# "solved" (default): the synthetic theta path (problems.synthetic_sequence: theta_0 plus a
# small seeded drift per system) with x_hat_i = the device L-BFGS minimiser of every sample's
# lower problem at theta_i (sequence.solve_path, gradient norm SOLVE_GTOL, warm-started) --
# real lower-level solutions, so H and g = x_hat - x_true are what a bilevel run sees.  It is
# made for the WHOLE batch once per box on cuda:0, cached as a krecycle-sequence-v1 directory
# under .seqcache/ and loaded by every arm and rank (identical inputs for the GPU arm, the
# cpu_baseline leg and --impl reference).  "recorded": the reference's record_sequence
# pattern (device gradient descent with Armijo line searches; slow at these configs, whose
# hypergradients are O(1e4) at theta_0).  "synthetic": xhat = x_true + a smooth 3 % field.

SEQ_SYSTEMS = 16
# lower-level gradient-norm target per config: C1's 1e-8 is BASELINE's; below ~1e-6 (C2/C3) or
# ~1e-4 (C4: cost ~1e5, 16 x 512^2) the Armijo test sits in the cost's roundoff and backtracks
# 30 times per iteration (the reference algorithm does the same)
SOLVE_GTOLS = {"C1": 1e-8, "C2": 1e-6, "C3": 1e-6, "C4": 1e-4, "C5": 1e-5}
SOLVE_GTOL = 1e-6
REC_GTOL, REC_BETA0, REC_DELTA = 1e-6, 1e-5, 1e-8


def sequence_dir(name: str, kind: str, systems: int) -> Path:
    tag = f"gtol{SOLVE_GTOLS.get(name, SOLVE_GTOL):g}" if kind == "solved" else f"gtol{REC_GTOL:g}_beta{REC_BETA0:g}"
    return ROOT / ".seqcache" / f"{name}_{kind}_sys{systems}_{tag}"


def ensure_sequence(args, systems: int):
    """Path of the workload's frozen sequence (made on cuda:0 if not cached); None for the
    synthetic sequence."""
    if args.sequence == "synthetic":
        return None
    if args.sequence not in ("solved", "recorded"):
        return Path(args.sequence)
    systems = max(systems, SEQ_SYSTEMS)
    path = sequence_dir(args.config, args.sequence, systems)
    if (path / "manifest.json").exists():
        return path
    import torch

    from paper_2412_08264_b200.lower import LinesearchParams
    from paper_2412_08264_b200.problems import CONFIGS, sample_arrays, synthetic_sequence
    from paper_2412_08264_b200.sequence import record, save_sequence, solve_path

    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    with torch.cuda.device(0):
        if args.sequence == "solved":
            thetas, _ = synthetic_sequence(cfg, sample_arrays(cfg, 0)[0][None], systems, seed=1234)
            seq = solve_path(cfg, thetas, lower_gtol=SOLVE_GTOLS.get(args.config, SOLVE_GTOL))
        else:
            seq = record(cfg, systems, lower_gtol=REC_GTOL, delta=REC_DELTA,
                         linesearch=LinesearchParams(beta=REC_BETA0))
    tmp = path.with_name(path.name + f".tmp{os.getpid()}")
    save_sequence(seq, tmp)
    if not path.exists():
        os.replace(tmp, path)
    print(f"bench: {args.sequence} sequence of {args.config}, {systems} systems, made in "
          f"{time.perf_counter() - t0:.1f} s -> {path}", file=sys.stderr, flush=True)
    return path


def sequence_text(path) -> str:
    if path is None:
        return "synthetic frozen sequence (problems.synthetic_sequence: theta drift, xhat = x_true + smooth field)"
    rel = path.relative_to(ROOT) if str(path).startswith(str(ROOT)) else path
    if "_solved_" in path.name:
        return (f"frozen sequence {rel} (krecycle-sequence-v1): the synthetic theta path with xhat_i = the "
                f"device L-BFGS minimiser of every sample's lower problem at theta_i (gradient norm "
                f"{path.name.split('gtol')[-1]}, warm-started; sequence.solve_path)")
    return (f"recorded frozen sequence {rel} (krecycle-sequence-v1; recycling-free bilevel run recorded on "
            f"the device: batched L-BFGS to gradient norm {REC_GTOL:g}, Armijo upper steps from theta_0 with "
            f"initial step {REC_BETA0:g}, hypergradients by RMINRES to residual {REC_DELTA:g})")


def load_systems(path, first: int, count: int, systems: int):
    """(thetas, xhats [systems][count][n]) of samples [first, first + count) of a recorded sequence
    (only those samples' rows are read)."""
    import json as _json

    man = _json.loads((Path(path) / "manifest.json").read_text())
    B, n = int(man["batch"]), int(man["n"])
    if man["num_systems"] < systems:
        raise ValueError(f"{path}: {man['num_systems']} systems recorded, {systems} needed")
    if first + count > B:
        raise ValueError(f"{path}: samples [{first}, {first + count}) beyond its batch of {B}")
    arr = Path(path) / "arrays"
    thetas, xhats = [], []
    for m in man["systems"][:systems]:
        tag = f"{m['index']:03d}"
        thetas.append(np.fromfile(arr / f"theta_{tag}.f64", dtype="<f8"))
        xhats.append(np.fromfile(arr / f"xhat_{tag}.f64", dtype="<f8", count=count * n,
                                 offset=first * n * 8).reshape(count, n))
    return thetas, xhats


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, _lib
    from paper_2412_08264_b200.bilevel import hypergradients
    from paper_2412_08264_b200.distributed import allgather_sum
    from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    first, B, total = samples_for(args.config, cfg, world, rank)
    model = make_batch(cfg, first=first, count=B)
    n = model.n
    steps_total = args.warmup + args.steps
    xt = model.x_true.cpu().numpy()
    # the frozen sequence: recorded once (rank 0 records the whole batch; the others wait)
    seq_path = None
    if rank == 0:
        seq_path = ensure_sequence(args, steps_total)
    if world > 1:
        obj = [None if seq_path is None else str(seq_path)]
        dist.broadcast_object_list(obj, src=0)
        seq_path = None if obj[0] is None else Path(obj[0])
    if seq_path is None:
        thetas, xhats_np = synthetic_sequence(cfg, xt, steps_total, seed=1234, first=first)
    else:
        thetas, xhats_np = load_systems(seq_path, first, B, steps_total)
    xhats = [torch.as_tensor(x, device="cuda") for x in xhats_np]
    solver_cfg = HessianSolveConfig.from_strategy(args.strategy, recycle_dim=cfg.recycle_dim, delta=args.delta,
                                                  method=cfg.method, max_iter=cfg.max_iter)

    def step(seq, i, X):
        hg, res, rec = hypergradients(model, thetas[i], X, seq)
        d = allgather_sum(hg, total)  # sample-ordered sum, bitwise equal for any world size
        return d, res

    # reserve the caching allocator's pool up front so per-step shape changes (t grows
    # with the previous solve's iteration count) do not hit cudaMalloc inside the timed region
    t_max = cfg.max_iter + cfg.recycle_dim
    per_sample = 8 * n * t_max * 6  # W, H W, candidates, QR workspaces of one sample's recycle update
    # Per-stream pools cannot lend memory to each other: when the job's working set (bases,
    # recycle state, update scratch: ~12 n t_max doubles per sample) is a large part of the device
    # (C4: 16 x 512^2 x 540), pre-sizing the pools would strand memory on the wrong streams; the
    # warm-up steps grow the pools instead.
    total_mem = torch.cuda.get_device_properties(local).total_memory
    seq = SequenceSolver(solver_cfg)
    if B * 12 * 8 * n * t_max < 0.35 * total_mem:
        torch.empty(3 * 1024**3 // 8, dtype=torch.float64, device="cuda")
        seq.reserve(B, per_sample, shape=(n, t_max))
    for i in range(args.warmup):
        step(seq, i, xhats[i])
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.LAUNCHES.clear()
    _lib.PROFILE = []
    evs, iters = [], []
    gc.collect()  # no cyclic-GC pauses inside timed regions
    gc.disable()
    clk = ClockSampler(local)
    dbg = os.environ.get("KR_BENCH_DEBUG")
    with clk:
        for i in range(args.warmup, steps_total):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            d, res = step(seq, i, xhats[i])
            e1.record()
            evs.append((e0, e1))
            iters.append([r.iterations for r in res])
            if dbg:
                torch.cuda.synchronize()
                print(f"step {i}: {e0.elapsed_time(e1):.1f} ms iters {iters[-1]}", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gc.enable()
    launches = _lib.total_launches()
    prof = _lib.PROFILE
    _lib.PROFILE = None
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    hg_count = total * args.steps
    value = hg_count / (total_ms / 1e3)

    # roofline of the dominant kernel (the persistent RMINRES / recycled-CG solve)
    kname = "kr_cg" if cfg.method == "cg" else "kr_rminres"
    wts = 3 if cfg.reg == "tv" else cfg.num_filters
    k_ms, k_bytes, k_iters, k_launch = 0.0, 0.0, 0, 0
    for a, b, info in prof:
        if info["kernel"] != kname:
            continue
        k_ms += a.elapsed_time(b)
        its = int(info["iters"].sum().item())
        k_iters += its
        k_launch += 1
        k_bytes += its * krylov_bytes_per_iter(kname, info["n"], info["s"], info["nsc"], wts)
    peak, peak_src = measured_peak()
    achieved = (k_bytes / 1e9) / (k_ms / 1e3) if k_ms > 0 else 0.0
    traffic = measured_traffic(args.config, kname)
    bytes_per_iter = k_bytes / max(k_iters, 1)
    traffic_per_launch = None
    if traffic is not None and traffic[2]:
        # the capture's DRAM bytes per batched iteration x this run's iterations per launch
        traffic_per_launch = traffic[0] / traffic[2] * (k_iters / max(k_launch, 1))

    hvp_line = hvp_fp64_roofline(model, thetas[-1], xhats[-1], cfg) if rank == 0 else None

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(x).pin_memory() for x in xhats_np]
        # the timed run's solver state (bases, recycle spaces, update scratch: ~100 GB at C4) is
        # released before the e2e pass builds its own
        del seq
        gc.collect()
        torch.cuda.empty_cache()
        seq2 = SequenceSolver(solver_cfg)
        if B * 12 * 8 * n * t_max < 0.35 * total_mem:
            seq2.reserve(B, per_sample, shape=(n, t_max))
        for i in range(args.warmup):
            X = pinned[i].to("cuda", non_blocking=True)
            step(seq2, i, X)[0].cpu()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        for i in range(args.warmup, steps_total):
            X = pinned[i].to("cuda", non_blocking=True)
            d, _ = step(seq2, i, X)
            d.cpu()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        gc.enable()
        if world > 1:
            t = torch.tensor([wall], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        e2e = {"value": hg_count / wall, "unit": "hypergradients/s",
               "h2d_bytes_per_step": int(B * n * 8), "d2h_bytes_per_step": int(model.num_params * 8)}

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_baseline(args)
    if rank == 0:
        flat_iters = [x for row in iters for x in row]
        line = {
            "metric": METRIC, "value": value, "unit": "hypergradients/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": {"strong": "strong", "weak": "weak", "replica": "weak"}[SHARDING.get(args.config, "weak")],
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_text(args.config, cfg, B, total, args),
                       "samples_total": total, "samples_per_gpu": B, "image": cfg.size,
                       "recycle_dim": cfg.recycle_dim, "max_iter": cfg.max_iter, "strategy": args.strategy,
                       "delta": args.delta, "krylov": cfg.method,
                       "sequence": sequence_text(seq_path),
                       "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"sample-sharded dp{world} ({SHARDING.get(args.config, 'weak')})"},
            "step_ms": [round(x, 3) for x in step_ms],
            "iterations_per_solve": {"mean": float(np.mean(flat_iters)), "min": int(np.min(flat_iters)),
                                     "max": int(np.max(flat_iters)), "at_max_iter": int(np.sum(
                                         np.asarray(flat_iters) >= cfg.max_iter))},
            "roofline": {"kernel": f"{kname} (persistent {'recycled CG' if kname == 'kr_cg' else 'RMINRES'}, "
                                   "all iterations of all samples)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None,
                         "traffic": traffic_per_launch,
                         "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum "
                                         "per batched iteration of the capture x this run's iterations per launch)",
                         "traffic_source": None if traffic is None else traffic[1],
                         "algorithmic_bytes_per_launch": k_bytes / max(k_launch, 1),
                         "algorithmic_bytes_per_iteration": bytes_per_iter,
                         "peak_source": peak_src,
                         "algorithmic_bytes": ("per iteration per sample 8n(12+3s+s_nsc)+8n*w (recycled CG)"
                                               if kname == "kr_cg" else
                                               "SURVEY 8(d): per iteration per sample 8n(21+3s+s_nsc)+8n(2+J)"),
                         "kernel_ms_total": k_ms, "kernel_share_of_step": k_ms / total_ms if total_ms else None,
                         "krylov_iterations": k_iters},
            "hvp_fp64": hvp_line,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "e2e": e2e,
            "cpu_baseline": cpu_base,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def hvp_fp64_roofline(model, theta, xhat, cfg, cols: int = 64):
    """The H W product of the recycle update (kr_hvp over `cols` columns of every sample)
    timed alone with CUDA events, against the measured fp64 peak: SURVEY 8(d)'s
    n F flops per column (F = 8b + J(4q^2 + 2) + 2)."""
    import torch

    H, _ = model.at(theta, xhat)
    B, n = model.batch, model.n
    W = torch.randn(B, cols, n, dtype=torch.float64, device="cuda").transpose(1, 2)  # (B, n, t), columns contiguous
    for _ in range(2):
        H._apply_cols(W)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        H._apply_cols(W)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = B * cols * n * hvp_flops_per_pixel(cfg)
    peak, src = measured_fp64_peak()
    achieved = flops / (ms / 1e3) / 1e12
    return {"kernel": "hvp_kernel (H W of the recycle update)", "bound": "fp64", "columns": B * cols,
            "ms": ms, "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "flops_per_pixel": hvp_flops_per_pixel(cfg), "peak_source": src}


# ---------------------------------------------------------------------------
# CPU legs: the oracle port of the reference algorithm (oracle/ restates krecycle's
# SequenceSolver / rminres / next_recycle / NscRule with the config operators).  Worker
# processes are started with the spawn method AFTER the BLAS thread variables are set, so
# each one imports numpy single-threaded.


def _cpu_worker(conn, name, k, strategy, delta, seq_path=None):
    """Owns sample k's oracle SequenceSolver; runs the systems it is sent, returns wall times."""
    from oracle import cpu_bilevel as ob
    from oracle import cpu_imaging as im
    from paper_2412_08264_b200.problems import CONFIGS, sample_arrays, synthetic_sequence

    cfg = CONFIGS[name]
    x_true, y = sample_arrays(cfg, k)
    taps = im.gaussian_taps(cfg.blur_size, cfg.blur_sigma)
    data = im.DataTerm("blur", (cfg.size, cfg.size), y, scale=2.0, ridge=0.0, taps=taps, x_true=x_true)
    reg = (im.Regularizer("filters", cfg.num_filters, cfg.kernel_size, "smooth_abs", cfg.eps) if cfg.reg != "tv"
           else im.Regularizer("tv", eps=cfg.eps))
    model = im.Model(data, reg)
    solver = ob.SequenceSolver(ob.SolveConfig.from_strategy(strategy, recycle_dim=cfg.recycle_dim, delta=delta,
                                                            max_iter=cfg.max_iter, method=cfg.method))
    thetas = xhats = None
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            break
        i, steps = msg
        if thetas is None or len(thetas) < steps:
            if seq_path is None:
                thetas, xs = synthetic_sequence(cfg, x_true[None], steps, seed=1234, first=k)
            else:
                thetas, xs = load_systems(seq_path, k, 1, steps)
            xhats = [x[0] for x in xs]
        t0 = time.perf_counter()
        H = im.hessian(model, thetas[i], xhats[i])
        J = im.jacobian(model, thetas[i], xhats[i])
        res, _ = solver.solve(H, xhats[i] - x_true, J)
        J.apply_adjoint(res.solution)
        conn.send((res.iterations, time.perf_counter() - t0))


def _spawn_workers(name, samples, strategy, delta, seq_path=None):
    import multiprocessing as mp

    for v in THREAD_ENV:
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    conns, procs = [], []
    for k in samples:
        parent, child = ctx.Pipe()
        pr = ctx.Process(target=_cpu_worker, args=(child, name, k, strategy, delta, seq_path), daemon=True)
        pr.start()
        conns.append(parent)
        procs.append(pr)
    for c in conns:
        assert c.recv() == "ready"
    return conns, procs


def _run_cpu(name, samples, strategy, delta, steps_cap, budget, seq_path=None):
    """System 0 (cold, untimed), then recycled systems 1, 2, ... on every worker in parallel
    until steps_cap systems or `budget` seconds of timed work (at least one system)."""
    conns, procs = _spawn_workers(name, samples, strategy, delta, seq_path)
    total_systems = steps_cap + 1

    def one(i):
        for c in conns:
            c.send((i, total_systems))
        return [c.recv() for c in conns]

    one(0)
    t0 = time.perf_counter()
    done, its = 0, []
    while done < steps_cap:
        its += [r[0] for r in one(1 + done)]
        done += 1
        if time.perf_counter() - t0 >= budget:
            break
    dt = time.perf_counter() - t0
    for c in conns:
        c.send(None)
    for pr in procs:
        pr.join(timeout=30)
    return done, dt, its


def cpu_baseline(args):
    """The oracle port on ONE host core (a spawned single-threaded process), sample 0:
    system 0 untimed, then recycled systems until --cpu-budget seconds."""
    seq_path = ensure_sequence(args, args.warmup + args.steps)
    done, dt, its = _run_cpu(args.config, [0], args.strategy, args.delta, max(args.steps, 1), args.cpu_budget,
                             seq_path)
    return {"value": done / dt, "unit": "hypergradients/s", "cores": 1, "kind": "port",
            "sample": f"sample 0, recycled systems 1..{done} after an untimed cold system 0 ({done} hypergradients, "
                      f"{dt:.1f} s, iterations {its}); single-threaded BLAS in a spawned process"}


def run_reference(args):
    """The reference's CPU path: the oracle port of krecycle's SequenceSolver / rminres /
    next_recycle / NscRule with the config's operators, one single-threaded process per
    host core, each owning one sample's recycling state (samples 0..cores-1 of the
    config's N=1 workload).  Bounded: one untimed cold system, then recycled systems
    until --steps or --ref-budget seconds.  Under torchrun only rank 0 runs."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2412_08264_b200.problems import CONFIGS

    cfg = CONFIGS[args.config]
    _, count, _ = samples_for(args.config, cfg, 1, 0)
    cores = len(os.sched_getaffinity(0))
    nproc = max(1, min(cores, count))
    seq_path = ensure_sequence(args, args.warmup + args.steps)
    done, dt, its = _run_cpu(args.config, list(range(nproc)), args.strategy, args.delta, max(args.steps, 1),
                             args.ref_budget, seq_path)
    value = nproc * done / dt
    line = {
        "metric": METRIC, "impl": "reference",
        "value": value, "unit": "hypergradients/s", "n_gpus": world, "steps": done, "warmup": 1,
        "ms_per_step": 1e3 * dt / done, "higher_is_better": True,
        "scaling": {"strong": "strong", "weak": "weak", "replica": "weak"}[SHARDING.get(args.config, "weak")],
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_text(args.config, cfg, count, count, args),
                   "bounded": f"samples 0..{nproc - 1} ({nproc} of {count}; one process per core), "
                              f"recycled systems 1..{done} timed after an untimed cold system 0 "
                              f"(--steps {args.steps}, budget {args.ref_budget:.0f} s)",
                   "strategy": args.strategy, "delta": args.delta, "iterations_mean": float(np.mean(its)),
                   "sequence": sequence_text(seq_path)},
        "cpu_baseline": {"value": value, "unit": "hypergradients/s", "cores": nproc, "kind": "port",
                         "sample": f"{nproc} samples x {done} recycled systems, one single-threaded process per core"},
        "e2e": {"value": value, "unit": "hypergradients/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    relaunch_if_needed(a)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)

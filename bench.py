"""Benchmark: hypergradients/sec of the recycled hypergradient solve (BASELINE.json metric).

A "step" is one upper-level system of the replay protocol (experiments.py:390-463)
for every sample of the batch: next_recycle (RGen-L(R): candidate basis, H W,
J W, projected GSVD, prepare_recycle) + the batched recycled-MINRES solve with
the NSC stop rule + J w, summed over samples (and over ranks for N > 1).

Workload (N=1): BASELINE configs[1] ("C2"): 8 samples of 128x128, blur 9x9
sigma 1.5, 1% noise, J=8 learned 5x5 filters (p=208), phi_eps eps=1e-2,
recycle dimension 20, max 200 Krylov iterations, NSC tolerance 1e-6.
Inputs: seeded synthetic (problems.py); the frozen sequence of systems is
synthetic (theta drifting, xhat = x_true + slowly drifting smooth field).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun): weak scaling, each rank owns its own 8 samples
(seeds offset by rank); the per-rank hypergradient sums are all-reduced.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

# load every CUDA module at context creation: a library kernel first used inside
# the timed region (e.g. the Householder rank-drop path) must not pay module loading there
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

STRATEGY = "RGen-L(R)-NSC"
DELTA = 1e-6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--strategy", default=STRATEGY)
    ap.add_argument("--delta", type=float, default=DELTA)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


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


def measured_traffic(config: str, kernel: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/r1_traffic.json), or None when this config/kernel was not captured."""
    p = Path(__file__).resolve().parent / "profiles" / "r1_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(config)
    if not d or d.get("kernel") != kernel:
        return None
    return int(d["dram_bytes_per_launch"]), d.get("source")


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


# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, _lib
    from paper_2412_08264_b200.bilevel import hypergradients
    from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    B = cfg.batch
    model = make_batch(cfg, first=rank * B, count=B)
    n = model.n
    steps_total = args.warmup + args.steps
    xt = model.x_true.cpu().numpy()
    thetas, xhats_np = synthetic_sequence(cfg, xt, steps_total, seed=1234 + rank)
    xhats = [torch.as_tensor(x, device="cuda") for x in xhats_np]
    solver_cfg = HessianSolveConfig.from_strategy(args.strategy, recycle_dim=cfg.recycle_dim, delta=args.delta,
                                                  method=cfg.method,
                                                  max_iter=cfg.max_iter)

    from paper_2412_08264_b200.distributed import allgather_sum

    def step(seq, i, X):
        hg, res, rec = hypergradients(model, thetas[i], X, seq)
        d = allgather_sum(hg, B * world)  # sample-ordered sum, bitwise equal for any world size
        return d, res

    # ---- device-resident run: warmup + timed ----
    # reserve the caching allocator's pool up front so per-step shape changes (t grows
    # with the previous solve's iteration count) do not hit cudaMalloc inside the timed region
    torch.empty(3 * 1024**3 // 8, dtype=torch.float64, device="cuda")
    t_max = cfg.max_iter + cfg.recycle_dim
    per_sample = 8 * n * t_max * 6  # W, H W, candidates, QR workspaces of one sample's recycle update
    seq = SequenceSolver(solver_cfg)
    seq.reserve(B, per_sample, shape=(n, t_max))
    for i in range(args.warmup):
        step(seq, i, xhats[i])
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.LAUNCHES.clear()
    _lib.PROFILE = []
    evs = []
    iters = []
    # no cyclic-GC pauses inside timed regions (collect now, re-enable afterwards)
    gc.collect()
    gc.disable()
    clk = ClockSampler(local)
    with clk:
        dbg = os.environ.get("KR_BENCH_DEBUG")
        if dbg:
            from paper_2412_08264_b200 import batched as _bt
            _bt.STATS = {}
            if dbg == "mem":  # stack traces of every caching-allocator segment allocation
                torch.cuda.memory._record_memory_history(max_entries=200000)
        for i in range(args.warmup, steps_total):
            if dbg:
                m0 = torch.cuda.memory_stats()
                s0 = dict(_bt.STATS)
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            d, res = step(seq, i, xhats[i])
            e1.record()
            evs.append((e0, e1))
            iters.append([r.iterations for r in res])
            if dbg:
                torch.cuda.synchronize()
                m1 = torch.cuda.memory_stats()
                ds = {k: _bt.STATS[k] - s0.get(k, 0) for k in _bt.STATS}
                if dbg == "mem" and m1.get('num_device_alloc', 0) > m0.get('num_device_alloc', 0):
                    snap = torch.cuda.memory._snapshot()
                    for tr in snap.get("device_traces", [[]])[0]:
                        if tr.get("action") == "segment_alloc":
                            fr = [f"{f['filename'].split('/')[-1]}:{f['line']}:{f['name']}" for f in tr.get("frames", [])
                                  if "paper_2412" in f["filename"] or "bench" in f["filename"]]
                            print(f"  segment_alloc {tr['size']} stream {tr.get('stream')} {fr[:6]}", file=sys.stderr)
                    torch.cuda.memory._record_memory_history(enabled=None)
                    torch.cuda.memory._record_memory_history(max_entries=200000)
                print(f"step {i}: {e0.elapsed_time(e1):.1f} ms iters {iters[-1]} stats {ds} "
                      f"mallocs {m1.get('num_device_alloc', 0) - m0.get('num_device_alloc', 0)} "
                      f"retries {m1.get('num_alloc_retries', 0) - m0.get('num_alloc_retries', 0)}",
                      file=sys.stderr, flush=True)
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
    hg_count = B * args.steps * world
    value = hg_count / (total_ms / 1e3)

    # roofline of the dominant kernel (the persistent RMINRES / recycled-CG solve)
    kname = "kr_cg" if cfg.method == "cg" else "kr_rminres"
    wts = 3 if cfg.reg == "tv" else cfg.num_filters
    k_ms, k_bytes, k_iters = 0.0, 0.0, 0
    for a, b, info in prof:
        if info["kernel"] != kname:
            continue
        ms = a.elapsed_time(b)
        its = int(info["iters"].sum().item())
        k_ms += ms
        k_iters += its
        k_bytes += its * krylov_bytes_per_iter(kname, info["n"], info["s"], info["nsc"], wts)
    peak, peak_src = measured_peak()
    achieved = (k_bytes / 1e9) / (k_ms / 1e3) if k_ms > 0 else 0.0
    traffic = measured_traffic(args.config, kname)

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(x).pin_memory() for x in xhats_np]
        seq2 = SequenceSolver(solver_cfg)
        seq2.reserve(B, per_sample, shape=(n, t_max))
        for i in range(args.warmup):
            X = pinned[i].to("cuda", non_blocking=True)
            step(seq2, i, X).__getitem__(0).cpu()
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
        cpu_base = cpu_baseline(cfg, xt, thetas, xhats_np, args)
    if rank == 0:
        flat_iters = [x for row in iters for x in row]
        line = {
            "metric": "hypergradients/sec (recycled solve incl. HVP) + achieved HBM GB/s vs peak",
            "value": value, "unit": "hypergradients/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {B} samples x {cfg.size}^2, blur {cfg.blur_size} "
                                   f"sigma {cfg.blur_sigma}, J={cfg.num_filters} q={cfg.kernel_size}, "
                                   f"s={cfg.recycle_dim}, max {cfg.max_iter} it, {args.strategy} delta={args.delta}, "
                                   f"{'recycled CG' if cfg.method == 'cg' else 'RMINRES'}",
                       "samples_per_gpu": B, "image": cfg.size, "recycle_dim": cfg.recycle_dim,
                       "max_iter": cfg.max_iter, "strategy": args.strategy, "delta": args.delta,
                       "krylov": cfg.method,
                       "sequence": "synthetic frozen sequence (problems.synthetic_sequence)",
                       "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"sample-sharded dp{world}"},
            "step_ms": [round(x, 3) for x in step_ms],
            "iterations_per_solve": {"mean": float(np.mean(flat_iters)), "min": int(np.min(flat_iters)),
                                     "max": int(np.max(flat_iters))},
            "roofline": {"kernel": f"{kname} (persistent {'recycled CG' if kname == 'kr_cg' else 'RMINRES'}, "
                                   "all iterations of all samples)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None,
                         "traffic": None if traffic is None else traffic[0],
                         "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                         "traffic_source": None if traffic is None else traffic[1],
                         "algorithmic_bytes_per_launch": (k_bytes / max(len([1 for _, _, i in prof
                                                                            if i["kernel"] == kname]), 1)),
                         "peak_source": peak_src,
                         "algorithmic_bytes": ("per iteration per sample 8n(12+3s+s_nsc)+8n*w (recycled CG)"
                                               if kname == "kr_cg" else
                                               "SURVEY 8(d): per iteration per sample 8n(21+3s+s_nsc)+8n(2+J)"),
                         "kernel_ms_total": k_ms, "kernel_share_of_step": k_ms / total_ms if total_ms else None,
                         "krylov_iterations": k_iters},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "e2e": e2e,
            "cpu_baseline": cpu_base,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _oracle_solve_sample(payload):
    """One hypergradient of one sample through the CPU oracle (reference algorithm)."""
    from oracle import cpu_bilevel as ob
    from oracle import cpu_imaging as im

    cfg, k, x_true, y, thetas, xhats, strategy, delta, systems = payload
    taps = im.gaussian_taps(cfg.blur_size, cfg.blur_sigma)
    shape = (cfg.size, cfg.size)
    data = im.DataTerm("blur", shape, y, scale=2.0, ridge=0.0, taps=taps, x_true=x_true)
    reg = im.Regularizer("filters", cfg.num_filters, cfg.kernel_size, "smooth_abs", cfg.eps) if cfg.reg != "tv" \
        else im.Regularizer("tv", eps=cfg.eps)
    model = im.Model(data, reg)
    solver = ob.SequenceSolver(ob.SolveConfig.from_strategy(strategy, recycle_dim=cfg.recycle_dim, delta=delta,
                                                            max_iter=cfg.max_iter, method=cfg.method))
    count = 0
    for i in systems:
        H = im.hessian(model, thetas[i], xhats[i])
        J = im.jacobian(model, thetas[i], xhats[i])
        res, _ = solver.solve(H, xhats[i] - x_true, J)
        J.apply_adjoint(res.solution)
        count += 1
    return count


def cpu_baseline(cfg, xt, thetas, xhats_np, args):
    """The oracle port timed on this host, single core, bounded sample."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from paper_2412_08264_b200.problems import sample_arrays

    _, y = sample_arrays(cfg, 0)
    systems = [0, 1]
    t0 = time.perf_counter()
    cnt = _oracle_solve_sample((cfg, 0, xt[0], y, thetas, [x[0] for x in xhats_np], args.strategy, args.delta,
                                systems))
    dt = time.perf_counter() - t0
    return {"value": cnt / dt, "unit": "hypergradients/s", "cores": 1, "kind": "port",
            "sample": f"sample 0, systems 0-1 of the same frozen sequence ({cnt} hypergradients, {dt:.1f} s)"}


def _reference_worker(conn, payload):
    """Persistent CPU worker owning one sample's SequenceSolver (recycling state carries over)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import cpu_bilevel as ob
    from oracle import cpu_imaging as im

    cfg, k, x_true, y, thetas, xhats, strategy, delta = payload
    taps = im.gaussian_taps(cfg.blur_size, cfg.blur_sigma)
    data = im.DataTerm("blur", (cfg.size, cfg.size), y, scale=2.0, ridge=0.0, taps=taps, x_true=x_true)
    reg = im.Regularizer("filters", cfg.num_filters, cfg.kernel_size, "smooth_abs", cfg.eps) if cfg.reg != "tv" \
        else im.Regularizer("tv", eps=cfg.eps)
    model = im.Model(data, reg)
    solver = ob.SequenceSolver(ob.SolveConfig.from_strategy(strategy, recycle_dim=cfg.recycle_dim, delta=delta,
                                                            max_iter=cfg.max_iter, method=cfg.method))
    while True:
        i = conn.recv()
        if i is None:
            break
        H = im.hessian(model, thetas[i], xhats[i])
        J = im.jacobian(model, thetas[i], xhats[i])
        res, _ = solver.solve(H, xhats[i] - x_true, J)
        J.apply_adjoint(res.solution)
        conn.send(res.iterations)


def run_reference(args):
    """The reference's CPU path: the oracle port of krecycle's SequenceSolver / rminres /
    next_recycle / NscRule with the config's operators, one process per host core, each
    process owning one sample's recycling state across steps (same workload as ours,
    bounded to min(cores, batch) samples)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    from paper_2412_08264_b200.problems import CONFIGS, sample_arrays, synthetic_sequence

    cfg = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    nproc = max(1, min(cores, cfg.batch))
    data = [sample_arrays(cfg, k) for k in range(cfg.batch)]
    xt = np.stack([d[0] for d in data])
    warm = min(args.warmup, 1)
    steps_total = warm + args.steps
    thetas, xhats_np = synthetic_sequence(cfg, xt, args.warmup + args.steps, seed=1234)
    ctx = mp.get_context("fork")
    conns, procs = [], []
    for k in range(nproc):
        parent, child = ctx.Pipe()
        payload = (cfg, k, xt[k], data[k][1], thetas, [x[k] for x in xhats_np], args.strategy, args.delta)
        pr = ctx.Process(target=_reference_worker, args=(child, payload), daemon=True)
        pr.start()
        conns.append(parent)
        procs.append(pr)

    def one_step(i):
        for c in conns:
            c.send(i)
        return [c.recv() for c in conns]

    for i in range(warm):
        one_step(i)
    t0 = time.perf_counter()
    its = []
    for i in range(warm, steps_total):
        its += one_step(i)
    dt = time.perf_counter() - t0
    for c in conns:
        c.send(None)
    for pr in procs:
        pr.join(timeout=30)
    done = nproc * args.steps
    value = done / dt
    line = {
        "metric": "hypergradients/sec (recycled solve incl. HVP) + achieved HBM GB/s vs peak", "impl": "reference",
        "value": value, "unit": "hypergradients/s", "n_gpus": world, "steps": args.steps, "warmup": warm,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}, bounded to {nproc} of {cfg.batch} samples (one per core); "
                               f"systems {warm}..{steps_total - 1} timed, {warm} warm-up system",
                   "strategy": args.strategy, "delta": args.delta, "iterations_mean": float(np.mean(its))},
        "cpu_baseline": {"value": value, "unit": "hypergradients/s", "cores": nproc, "kind": "port",
                         "sample": f"{nproc} samples x {args.steps} recycled systems, one process per core"},
        "e2e": {"value": value, "unit": "hypergradients/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)

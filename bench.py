#!/usr/bin/env python
"""sFISTA throughput on B200 (BASELINE.json metric: Mpixel*iterations/s).

Workload (N=1): BASELINE configs[1] = cfg2 — 1024x1024 phantom (200 rect + 100 disks), 63x63
two-Gaussian PSF, reflective BC (Toeplitz+Hankel factors), r=5, lam=0.01, x>=0, 200 iterations.
Headline dtype float64 (the reference computes in fp64); the float32 variant of the same config is
reported under "variants". One step = one complete 200-iteration solve. N>1: independent replicas
(cfg2 does not shard), weak scaling, value = total Mpix*it/s over ranks, time = max over
ranks. Inputs are L2-resident during a solve by design (40 MB working set); L2 is flushed (256 MiB
write) between timed steps.

--impl reference: the CPU oracle port of kronblur's hot path (oracle/kronblur_port.py; the reference
is pure Python/numpy and cannot travel to the GPU box) on the host cores, threaded over column
blocks; each step = one cfg2 iteration. Rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = "cfg2"
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default=CFG)
    p.add_argument("--dtype", default="float64", choices=["float64", "float32"])
    p.add_argument("--no-variants", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--row-blocks", action="store_true",
                   help="cfg4/cfg5: row-block sharded solve even at N=1 (automatic for N>1)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def committed_traffic(config, dtype):
    """Per-kernel DRAM bytes (read + write) of one iteration's four pass kernels from the
    committed ncu capture of this config (profiles/traffic_<config>.json, written by
    tools/ncu_traffic.py from an `ncu --set full` run of tools/one_iter.py), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", f"traffic_{config}.json")
    try:
        with open(path) as f:
            per = json.load(f).get("_per_kernel", {}).get(dtype)
        return [int(k["dram_bytes"]) for k in per] if per else None
    except (OSError, ValueError, KeyError, TypeError):
        return None


def l2_note(cfg, dtype, images=1):
    esz = 8 if dtype == "float64" else 4
    ws = images * (4 + cfg.r) * cfg.m * cfg.m * esz / 1e6  # X, Y, B, R and the r Z planes
    where = "L2-resident within a solve" if ws < 100 else "larger than L2 (HBM-backed)"
    return f"flushed between steps (256 MiB write); {ws:.0f} MB working set is {where}"


def device_operator_batch(ops, dtype):
    from paper_1901_00913_b200.device import DeviceOperator

    return DeviceOperator(list(ops), dtype)


def algorithmic(cfg):
    """Per pixel*iteration: flops F = 8 r w (forward + adjoint, 2 passes each, w MACs per tap
    row), compulsory bytes 8*sizeof(T) (sweep 1 reads Y, B writes R; sweep 2 reads R, Y, X_prev,
    writes X, Y) — SURVEY §8(d)."""
    return 8 * cfg.r * cfg.w


def measured_peaks():
    try:
        with open(MEASURED) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        loaded = [s for s in sm if s is not None and s > 500] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": num(rows[0][1]), "reasons": reasons, "samples": len(rows)}


def build_problem(cfg, dtype, seed=0, device="cuda", images=None):
    """Seeded data, operator(s) and Lipschitz constant(s) of a config. Single-image configs give
    (B [m,m], op, L); batch configs (cfg3) give this rank's images (B [count,m,m], [op], [L])."""
    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200 import workloads as W

    if images is None:
        X, psf, B = W.make_image_data(cfg, seed=seed, device=device)
        op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
        L = kb.lipschitz(op, iters=50, seed=seed, dtype="float64")
        return B, op, L
    Bs, ops, Ls = [], [], []
    for i in images:  # each image has its own phantom and PSF (BASELINE cfg3)
        _, psf, B = W.make_image_data(cfg, seed=0, index=i, device=device)
        op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
        Bs.append(B)
        ops.append(op)
        Ls.append(kb.lipschitz(op, iters=50, seed=0, dtype="float64"))
    return np.stack(Bs), ops, np.array(Ls)


def run_b200(args):
    import torch

    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200 import workloads as W
    from paper_1901_00913_b200.device import INT_MAX, device_operator, fma_peak

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.CONFIGS[args.config]
    m, iters = cfg.m, cfg.iters

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    batched = cfg.batch > 1
    if batched:  # cfg3: the batch is sharded across ranks with no communication (strong scaling)
        from paper_1901_00913_b200.shard import batch_partition

        start, count = batch_partition(cfg.batch, world)[rank]
        B, ops, L = build_problem(cfg, args.dtype, images=range(start, start + count))
        op = ops[0]
    else:
        B, op, L = build_problem(cfg, args.dtype, seed=rank)
        ops = [op]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def measure(dtype, steps, warmup, clocks=False):
        from paper_1901_00913_b200.device import DeviceOperator

        dev = DeviceOperator(ops, dtype) if batched else device_operator(op, dtype)
        _, beta = kb.momentum_table(iters)
        Bd = torch.from_numpy(B).to("cuda", dev.tdtype)
        Xd, Yd = torch.zeros_like(Bd), torch.zeros_like(Bd)
        flag = torch.full((1,), INT_MAX, dtype=torch.int32, device="cuda")
        stream = torch.cuda.current_stream()
        times = []
        sampler = ClockSampler(local)
        for s in range(warmup + steps):
            Xd.zero_()
            Yd.zero_()
            flush.zero_()
            if s == warmup:
                barrier()
                torch.cuda.synchronize()
                if clocks:
                    sampler.__enter__()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dev.sfista_run(Bd, Xd, Yd, beta, 0, iters, L, cfg.lam, True, flag, use_graph=True)
            e1.record(stream)
            if s >= warmup:
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        barrier()
        if clocks:
            sampler.__exit__(None, None, None)
        assert int(flag.item()) > iters, "non-finite iterate in benchmark run"
        return dev, Bd, sum(times) / len(times), (sampler.summary() if clocks else None)

    dev, Bd, ms, clocks = measure(args.dtype, args.steps, args.warmup, clocks=True)
    ms = max_over_ranks(ms)
    mpix_it = m * m * iters / 1e6
    # whole-job units: every rank's images (batch) or one image per replica
    units = cfg.batch if batched else world
    value = units * mpix_it / (ms / 1e3)

    # ---- e2e: public API with host buffers (H2D of B, D2H of x inside the region; X0 = None)
    cfgsolve = kb.SolveConfig(lam=cfg.lam, lipschitz=float(np.max(L)), max_iter=iters, record_history=False)
    opts = kb.SolveOptions(dtype=args.dtype, project=True, use_graph=True)
    esz = 8 if args.dtype == "float64" else 4
    if batched:  # public batch API with host arrays: H2D of B, D2H of x inside the region
        dev_e2e = device_operator_batch(ops, args.dtype)

        def e2e_call():
            kb.sfista_batch(dev_e2e, B, L, cfg.lam, iters, options=opts)
    else:
        def e2e_call():
            kb.sfista(op, B, cfgsolve, options=opts)
    for _ in range(min(args.warmup, 3)):
        e2e_call()
    e2e_t = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e2e_call()
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(sum(e2e_t) / len(e2e_t))
    nimg = len(ops)
    e2e = {"value": units * mpix_it / e2e_s, "unit": "Mpixel*iterations/s",
           "h2d_bytes_per_step": nimg * m * m * esz,  # B (X0 = None is zeroed on the device)
           "d2h_bytes_per_step": nimg * m * m * esz}

    # ---- roofline of the dominant pass kernel (CUDA events on the launching stream)
    kern_ms = dev.time_passes(Bd, Bd, L, cfg.lam, reps=20)
    engines = dev.last_engines()
    it_ms = sum(kern_ms)
    F = algorithmic(cfg)
    flops_it = F * m * m * len(ops)
    # binding compute roof: the tensor instruction each pass issues, measured live. fp32 runs
    # 3xTF32 (three TF32 MMAs per fp32-accurate product), so its roof is the TF32 rate / 3.
    peak_of = {}

    def engine_peak(eng):
        if eng not in peak_of:
            if eng == "dmma":
                peak_of[eng] = (fma_peak("float64"), "FP64 tensor-core DMMA m8n8k4 burn")
            elif eng == "tcgen05_tf32":
                peak_of[eng] = (fma_peak("tcgen05_tf32") / 3.0,
                                "tcgen05.mma kind::tf32 M128 N256 K8 burn / 3 (3xTF32 passes)")
            else:  # mma.sync TF32 (and the FFMA / generic fallbacks, bounded by the same roof)
                peak_of[eng] = (fma_peak("float32") / 3.0, "TF32 tensor-core mma.sync m16n8k8 burn / 3 (3xTF32 passes)")
        return peak_of[eng]

    k_dom = max(range(4), key=lambda i: kern_ms[i])
    flops_pass = F / 4 * m * m * len(ops)  # one axis filter of all r terms over every pixel
    achieved_tf = flops_pass / (kern_ms[k_dom] * 1e-3) / 1e12
    peak_dom, peak_src = engine_peak(engines[k_dom])
    traffic = committed_traffic(cfg.name, args.dtype)
    peaks, peak_kind = measured_peaks()
    hbm_gbs = 8 * esz * m * m * len(ops) / (it_ms * 1e-3) / 1e9
    phase = ["pass A forward (split)", "pass B forward (sum, residual epilogue)",
             "pass A adjoint (split)", "pass B adjoint (sum, fused FISTA update)"]
    roofline = {
        "bound": "tensor",
        "kernel": f"{phase[k_dom]} on {engines[k_dom]}: the longest of the iteration's four kernels",
        "achieved": round(achieved_tf, 3), "peak": round(peak_dom, 3), "unit": "TFLOP/s",
        "frac": round(achieved_tf / peak_dom, 4),
        "peak_source": "measured live by kb_fma_peak in this run: " + peak_src,
        "traffic": traffic[k_dom] if traffic else None,
        # compulsory bytes of that launch: split reads X, writes r planes; residual sum reads r
        # planes + B, writes R; update sum reads r planes + Y + X_prev, writes X, Y
        "traffic_algorithmic_bytes": esz * m * m * len(ops) * (1 + cfg.r, cfg.r + 2, 1 + cfg.r, cfg.r + 4)[k_dom],
        "iteration": {
            "per_kernel_ms": [round(x, 5) for x in kern_ms],
            "engines": engines,
            "achieved": round(flops_it / (it_ms * 1e-3) / 1e12, 3),
            "frac_of_peak": [round(F / 4 * m * m * len(ops) / (t * 1e-3) / 1e12 / engine_peak(e)[0], 4)
                             for t, e in zip(kern_ms, engines)],
        },
        "hbm": {"achieved": round(hbm_gbs, 1), "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": round(hbm_gbs / peaks.get("hbm_gbs", 6550.0), 4), "peak_source": peak_kind,
                "algorithmic_bytes_per_px_it": 8 * esz},
        "algorithmic_flops_per_px_it": F,
        # taps the kernels execute per axis after trimming entries below 1e-14 of a generator's
        # peak; narrower than w when the PSF is ~0 near its window edges (cfg5's
        # motion line), in which case achieved (counted with the nominal w) can exceed the roof
        "executed_taps": [dev.bands[1], dev.bands[3]],
    }

    variants = {}
    if not args.no_variants and world == 1 and "float32" in cfg.dtypes and args.dtype != "float32":
        _, _, ms32, _ = measure("float32", max(2, args.steps // 2), 2)
        variants["float32"] = {"value": units * mpix_it / (ms32 / 1e3), "ms_per_step": ms32}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, op, B[0] if batched else B, L[0] if batched else L, iters_sample=2)

    if rank == 0:
        line = {
            "metric": "sFISTA Mpixel*iterations/s",
            "value": round(value, 2),
            "unit": "Mpixel*iterations/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 4),
            "higher_is_better": True,
            "scaling": "strong" if batched else "weak",
            "vs_baseline": None,
            "dtype": "f64" if args.dtype == "float64" else "f32",
            "data": f"synthetic (seeded phantom + PSF + exact-level Gaussian noise, BASELINE {cfg.name})",
            "config": {"workload": f"{args.config}: {(str(cfg.batch) + ' x ') if batched else ''}{m}x{m} "
                                   f"{cfg.bc} BC, w={cfg.w}, r={cfg.r}, lam={cfg.lam}, x>=0, "
                                   f"{iters} iterations per step",
                       "global_batch": cfg.batch if batched else world,
                       "parallelism": f"batch-shard{world}" if batched else f"replicas{world}",
                       "l2": l2_note(cfg, args.dtype, len(ops))},
            "e2e": e2e,
            "roofline": roofline,
            "gpu_launches": 4 * iters * args.steps,
            "clocks": clocks,
            "impl": "b200",
        }
        if variants:
            line["variants"] = variants
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_row_blocks(args):
    """cfg4 / cfg5 at N > 1 (or --row-blocks at N = 1): ONE image split into contiguous row blocks
    across ranks, shard.solve_row_blocks with two halo exchanges per iteration over
    NCCL (batch_isend_irecv). Strong scaling: value = m*m*iters of the whole image / max-over-ranks
    solve time. Every rank builds the same seeded problem and keeps its rows."""
    import torch

    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200 import workloads as W
    from paper_1901_00913_b200.device import fma_peak
    from paper_1901_00913_b200.shard import BlockPlan, DeviceBlockBackend, halo_rows, solve_row_blocks

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.CONFIGS[args.config]
    m, iters = cfg.m, cfg.iters
    B, op, L = build_problem(cfg, args.dtype, seed=0)
    plan = BlockPlan(m, m, world, rank, halo_rows(op))
    backend = DeviceBlockBackend(op, plan, args.dtype)
    tdt = torch.float64 if args.dtype == "float64" else torch.float32
    Bl = torch.from_numpy(np.ascontiguousarray(B[plan.g0:plan.g0 + plan.rows])).to("cuda", tdt)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.current_stream()
    times, sampler = [], ClockSampler(local)
    for s in range(args.warmup + args.steps):
        flush.zero_()
        if s == args.warmup:
            barrier()
            torch.cuda.synchronize()
            sampler.__enter__()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        solve_row_blocks(backend, plan, Bl, L, cfg.lam, iters, project=True)
        e1.record(stream)
        torch.cuda.synchronize()
        if s >= args.warmup:
            times.append(e0.elapsed_time(e1))
    barrier()
    sampler.__exit__(None, None, None)
    ms = max_over_ranks(sum(times) / len(times))
    value = m * m * iters / 1e6 / (ms / 1e3)

    # e2e: host rows in (pinned H2D), solve, x rows out, wall clock, max over ranks
    Bh = torch.from_numpy(np.ascontiguousarray(B[plan.g0:plan.g0 + plan.rows]).astype(
        np.float64 if args.dtype == "float64" else np.float32)).pin_memory()
    e2e_t = []
    for s in range(2 + args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Bd = Bh.to("cuda", non_blocking=True)
        x = solve_row_blocks(backend, plan, Bd, L, cfg.lam, iters, project=True).cpu()
        torch.cuda.synchronize()
        if s >= 2:
            e2e_t.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(sum(e2e_t) / len(e2e_t))
    esz = 8 if args.dtype == "float64" else 4
    eng = "tcgen05_tf32" if args.dtype == "float32" else "dmma"
    peak = fma_peak("tcgen05_tf32") / 3.0 if args.dtype == "float32" else fma_peak("float64")
    achieved = algorithmic(cfg) * m * m * iters / (ms * 1e-3) / 1e12 / world  # per GPU
    if rank == 0:
        line = {
            "metric": "sFISTA Mpixel*iterations/s", "value": round(value, 2), "unit": "Mpixel*iterations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.dtype == "float64" else "f32",
            "data": f"synthetic (seeded phantom + PSF + exact-level Gaussian noise, BASELINE {cfg.name})",
            "config": {"workload": f"{args.config}: {m}x{m} {cfg.bc} BC, w={cfg.w}, r={cfg.r}, lam={cfg.lam}, "
                                   f"x>=0, {iters} iterations per step, row blocks of {plan.rows} rows, "
                                   f"halo {plan.h}",
                       "global_batch": 1, "parallelism": f"row-blocks{world}",
                       "l2": "flushed between steps (256 MiB write); HBM-backed working set"},
            "e2e": {"value": m * m * iters / 1e6 / e2e_s, "unit": "Mpixel*iterations/s",
                    "h2d_bytes_per_step": m * m * esz, "d2h_bytes_per_step": m * m * esz},
            "roofline": {"bound": "tensor", "kernel": f"whole row-block iteration per GPU ({eng} passes, "
                                                      "halo exchanges included)",
                         "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4), "traffic": None},
            "gpu_launches": 4 * iters * args.steps,
            "clocks": sampler.summary(),
            "impl": "b200",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_baseline(cfg, op, B, L, iters_sample=2, threads=None):
    """Oracle port (kronblur's FFT hot path in numpy) on the host: a bounded sample of
    `iters_sample` projected iterations of the same workload."""
    from oracle import kronblur_port as port

    threads = threads or cpu_threads()
    pop = port.PortOperator(op)
    port.set_threads(threads)
    t0 = time.perf_counter()
    port.sfista(pop, B, L, cfg.lam, iters_sample, project=True)
    dt = time.perf_counter() - t0
    return {"value": round(cfg.m * cfg.m * iters_sample / dt / 1e6, 4), "unit": "Mpixel*iterations/s",
            "cores": threads, "kind": "port",
            "sample": f"{iters_sample} projected sFISTA iterations of {cfg.name} ({cfg.m}x{cfg.m}, fp64, "
                      f"numpy pocketfft path threaded over column blocks), {dt:.2f} s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_1901_00913_b200 as kb
    from oracle import kronblur_port as port
    from paper_1901_00913_b200 import workloads as W

    cfg = W.CONFIGS[args.config]
    X, psf, B = W.make_image_data(cfg, seed=0, device="cpu")
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
    threads = cpu_threads()
    port.set_threads(threads)
    pop = port.PortOperator(op)
    L = port.estimate_lipschitz(lambda v: port.kron_apply(pop, v),
                                lambda v: port.kron_apply_adjoint(pop, v), (cfg.m, cfg.m), 2, 0)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        port.sfista(pop, B, L, cfg.lam, 1, project=True)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    step = sum(times) / len(times)
    value = cfg.m * cfg.m / step / 1e6
    line = {
        "metric": "sFISTA Mpixel*iterations/s", "value": round(value, 4), "unit": "Mpixel*iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {cfg.name})",
        "config": {"workload": f"{args.config}: one projected sFISTA iteration per step on the CPU port",
                   "global_batch": 1, "parallelism": "cpu"},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpixel*iterations/s", "cores": threads,
                         "kind": "port", "sample": f"1 iteration of {cfg.name} per step"},
        "e2e": {"value": round(value, 4), "unit": "Mpixel*iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config in ("cfg4", "cfg5") and (args.row_blocks or dist_env()[1] > 1):
        run_row_blocks(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

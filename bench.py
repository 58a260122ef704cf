#!/usr/bin/env python
"""sFISTA throughput on B200 (BASELINE.json metric: Mpixel*iterations/s).

Headline workload (N=1): the largest single-GPU BASELINE config, cfg5 -- one 16384x16384 fp32
phantom (20000 rectangles + 10000 disks), 127x127 motion-line PSF, reflective BC
(Toeplitz+Hankel factors), r=10, lam=0.01, x>=0, 100 iterations. One step = one complete
100-iteration solve through the native loop (kb_sfista_run, one CUDA graph). cfg2 (fp64 and fp32),
cfg3 (512-image batch) and cfg4 are measured the same way under "variants" at N=1.

N>1 (`--gpus N`; bench.py re-executes itself under torch.distributed.run when WORLD_SIZE is
unset): cfg5 and cfg4 are row-block sharded (one image, contiguous row blocks per rank, halo
rows exchanged over NCCL) -- strong scaling, value = whole image Mpix*it/s over the
max-over-ranks solve time; cfg3 is batch sharded (no communication); cfg1/cfg2 run replicas.

--impl reference: the reference's CPU hot path (oracle/kronblur_port.py, the numpy pocketfft
restatement of kronblur; the reference is pure Python and cannot travel to the GPU box) on the
host cores, on the SAME config: each step times a bounded sample of one cfg5 iteration (one
Toeplitz+Hankel factor application of order m to a column block) and extrapolates it to the
whole iteration (4 r factor applications over all n columns). Rank 0 only.
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

CFG = "cfg5"
VARIANTS = (("cfg1", "float64"), ("cfg2", "float64"), ("cfg2", "float32"), ("cfg3", "float32"), ("cfg4", "float32"))
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default=CFG)
    p.add_argument("--dtype", default=None, choices=["float64", "float32"],
                   help="default: the config's first dtype (fp64 for cfg1/cfg2, fp32 otherwise)")
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


def committed_traffic(config, dtype, fused=False):
    """Per-kernel DRAM bytes (read + write) of one iteration's pass kernels from the committed
    ncu capture of this config (profiles/traffic_<config>.json, written by tools/ncu_traffic.py
    from an `ncu --set full` run of tools/one_iter.py), or None. With the one-sweep kernel the
    capture lists [forward, 0, adjoint, 0] under "_per_kernel_fused"."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", f"traffic_{config}.json")
    try:
        with open(path) as f:
            per = json.load(f).get("_per_kernel_fused" if fused else "_per_kernel", {}).get(dtype)
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


def build_problem(cfg, dtype, seed=0, device="cuda", images=None, lipschitz=True):
    """Seeded data, operator(s) and Lipschitz constant(s) of a config. Single-image configs give
    (B [m,m], op, L); batch configs (cfg3) give this rank's images (B [count,m,m], [op], [L]).
    lipschitz=False leaves L to the caller (None): the row-block path estimates it sharded."""
    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200 import workloads as W

    if images is None:
        X, psf, B = W.make_image_data(cfg, seed=seed, device=device)
        op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
        L = kb.lipschitz(op, iters=50, seed=seed, dtype="float64") if lipschitz else None
        return B, op, L
    Bs, ops, Ls = [], [], []
    for i in images:  # each image has its own phantom and PSF (BASELINE cfg3)
        _, psf, B = W.make_image_data(cfg, seed=0, index=i, device=device)
        op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
        Bs.append(B)
        ops.append(op)
        Ls.append(kb.lipschitz(op, iters=50, seed=0, dtype="float64"))
    return np.stack(Bs), ops, np.array(Ls)


def default_dtype(cfg):
    return cfg.dtypes[0]


def sustained_peak(kind, seconds=3.0):
    """(sustained, burst) rate of a tensor burn: the burn launched back to back for `seconds`
    (the median of the second half, once power capping has settled) and its first launch. The
    solve kernels run inside a long step, so their roofline divides by the sustained figure (the
    driver's rule for MEASURED_PEAKS.json: burst for a kernel timed alone, sustained for a kernel
    timed inside a long step)."""
    from paper_1901_00913_b200.device import fma_peak

    first = fma_peak(kind)
    vals, t0 = [], time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        vals.append(fma_peak(kind))
    tail = vals[len(vals) // 2:] or [first]
    return float(statistics.median(tail)), float(first)


def engine_peak(eng, cache={}):
    """Binding compute roof of a pass engine, measured live: the tensor instruction it issues
    (fp32 passes run 3xTF32, three TF32 MMAs per fp32-accurate product: TF32 rate / 3), sustained
    (sustained_peak)."""
    if eng not in cache:
        if eng == "dmma":
            sus, burst = sustained_peak("float64")
            cache[eng] = (sus, f"FP64 tensor-core DMMA m8n8k4 burn, sustained (burst {burst:.1f})")
        elif eng in ("tcgen05_tf32", "tcgen05_fused"):
            sus, burst = sustained_peak("tcgen05_tf32")
            cache[eng] = (sus / 3.0, f"tcgen05.mma kind::tf32 M128 N256 K8 burn / 3 (3xTF32 passes), sustained "
                                     f"(burst {burst / 3.0:.1f})")
        else:  # mma.sync TF32 (and the FFMA / generic fallbacks, bounded by the same roof)
            sus, burst = sustained_peak("float32")
            cache[eng] = (sus / 3.0, f"TF32 tensor-core mma.sync m16n8k8 burn / 3 (3xTF32 passes), sustained "
                                     f"(burst {burst / 3.0:.1f})")
    return cache[eng]


def launches_per_iteration(dev, engines=None):
    """Kernels of one fast-path iteration: 4 passes (one per direction where the one-sweep fused
    kernel runs it), plus the exact-fold kernels of a reflective axis whose generators are not
    (anti)symmetric (kb_capi.cu stage_a / stage_b)."""
    info = dev.info()
    if engines and engines[0] == "persist_f64":
        return 0  # counted per solve (one cooperative launch)
    n = 4 - sum(1 for i in (0, 2) if engines and engines[i] == "tcgen05_fused")
    if dev.bc[0] == 1 and not info["sym_a"]:
        n += 1
    if dev.bc[1] == 1 and not info["sym_b"]:
        n += 1
    return n


def measure_config(name, dtype, steps, warmup, rank, world, local, clocks=False, e2e_steps=None,
                   barrier=lambda: None, max_over_ranks=lambda x: x):
    """Time `steps` full solves of a config (inputs resident in HBM, L2 flushed between steps),
    then the same through the public API with host buffers (e2e), then the four pass kernels of
    one iteration (roofline). Returns the pieces of the JSON line."""
    import torch

    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200 import workloads as W
    from paper_1901_00913_b200.device import INT_MAX, DeviceOperator, device_operator

    cfg = W.CONFIGS[name]
    m, iters = cfg.m, cfg.iters
    batched = cfg.batch > 1
    if batched:  # cfg3: the batch is sharded across ranks with no communication (strong scaling)
        from paper_1901_00913_b200.shard import batch_partition

        start, count = batch_partition(cfg.batch, world)[rank]
        B, ops, L = build_problem(cfg, dtype, images=range(start, start + count))
        op = ops[0]
    else:
        B, op, L = build_problem(cfg, dtype, seed=rank)
        ops = [op]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
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
    engines_solve = dev.last_engines()
    ms = max_over_ranks(sum(times) / len(times))
    mpix_it = m * m * iters / 1e6
    units = cfg.batch if batched else world  # whole-job images
    value = units * mpix_it / (ms / 1e3)
    res = {"cfg": cfg, "dtype": dtype, "ms": ms, "value": value, "batched": batched, "ops": ops,
           "op": op, "B": B, "L": L, "clocks": sampler.summary() if clocks else None,
           "engines_solve": engines_solve,
           "launches": launches_per_iteration(dev, engines_solve) * iters * steps
           + (steps if engines_solve and engines_solve[0] == "persist_f64" else 0)}

    # ---- e2e: the public API with host buffers (H2D of B, D2H of x inside the region; X0 = None)
    esz = 8 if dtype == "float64" else 4
    if e2e_steps:
        opts = kb.SolveOptions(dtype=dtype, project=True, use_graph=True)
        if batched:
            def e2e_call():
                kb.sfista_batch(dev, B, L, cfg.lam, iters, options=opts)
        else:
            cfgsolve = kb.SolveConfig(lam=cfg.lam, lipschitz=float(L), max_iter=iters, record_history=False)

            def e2e_call():
                kb.sfista(op, B, cfgsolve, options=opts)
        e2e_call()
        t0 = time.perf_counter()
        e2e_call()
        torch.cuda.synchronize()
        if time.perf_counter() - t0 < 0.02:  # millisecond-scale calls (cfg1, cfg2): average more of them
            e2e_steps = max(e2e_steps, 20)
        e2e_t = []
        for _ in range(e2e_steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            e2e_call()
            torch.cuda.synchronize()
            e2e_t.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sum(e2e_t) / len(e2e_t))
        nimg = len(ops)
        # host arrays are fp64 (the reference API); they move as `dtype` through pinned pieces
        res["e2e"] = {"value": units * mpix_it / e2e_s, "unit": "Mpixel*iterations/s",
                      "h2d_bytes_per_step": nimg * m * m * esz, "d2h_bytes_per_step": nimg * m * m * esz,
                      "path": "public sfista / sfista_batch with host numpy B (fp64 in, fp64 x out)"}

    # ---- roofline of the dominant pass kernel (CUDA events on the launching stream)
    kern_ms = dev.time_passes(Bd, Bd, L, cfg.lam, reps=10 if m >= 8192 else 20)
    engines = dev.last_engines()
    wa, wb = dev.bands[1], dev.bands[3]  # executed taps per axis (band after trimming)
    px = m * m * len(ops)
    # one axis filter of all r terms per phase; with the axis-swapped twin (kb_capi.cu: the wider
    # band first) pass A filters axis 1 and pass B axis 0
    swapped = bool(dev.info().get("twin", 0))
    flops_phase = [2 * cfg.r * w * px for w in ((wb, wa, wb, wa) if swapped else (wa, wb, wa, wb))]
    # one-sweep fused directions (kb_fused.cuh): phase 0 / 2 is the whole application, 1 / 3 empty
    fused = [engines[2 * d] == "tcgen05_fused" for d in (0, 1)]
    for d in (0, 1):
        if fused[d]:
            flops_phase[2 * d] += flops_phase[2 * d + 1]
            flops_phase[2 * d + 1] = 0
    k_dom = max(range(4), key=lambda i: kern_ms[i])
    achieved_tf = flops_phase[k_dom] / (kern_ms[k_dom] * 1e-3) / 1e12
    peak_dom, peak_src = engine_peak(engines[k_dom])
    traffic = committed_traffic(cfg.name, dtype, fused=any(fused))
    peaks, peak_kind = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6550.0)
    it_ms = sum(kern_ms)
    phase = ["pass A forward (split)", "pass B forward (sum, residual epilogue)",
             "pass A adjoint (split)", "pass B adjoint (sum, fused FISTA update)"]
    if fused[0]:
        phase[0] = "forward application (one-sweep fused kernel, residual epilogue)"
    if fused[1]:
        phase[2] = "adjoint application (one-sweep fused kernel, FISTA update epilogue)"
    # DRAM bytes the dominant launch must move: two-sweep split reads X and writes r Z planes;
    # residual sum reads r Z planes + B, writes R; update sum reads r Z planes + Y + X_prev, writes
    # X and Y. The fused kernel keeps Z on chip: forward reads Y + B, writes R (3 planes); adjoint
    # reads R + Y + X_prev, writes X and Y (5 planes)
    per_phase = [1 + cfg.r, cfg.r + 2, 1 + cfg.r, cfg.r + 4]
    if fused[0]:
        per_phase[0], per_phase[1] = 3, 0
    if fused[1]:
        per_phase[2], per_phase[3] = 5, 0
    kern_bytes = esz * px * per_phase[k_dom]
    # Which roof binds the dominant kernel: its arithmetic intensity (flops on executed taps over
    # the DRAM bytes this two-sweep kernel must move, its r Z^T planes included) against the
    # machine balance (live tensor peak / measured HBM bandwidth). L2-resident configs (cfg1,
    # cfg2: the whole working set fits the 126 MB L2) are bounded by the tensor roof.
    ws_mb = len(ops) * (4 + cfg.r) * m * m * esz / 1e6
    intensity = flops_phase[k_dom] / kern_bytes
    balance = peak_dom * 1e12 / (hbm_peak * 1e9)
    hbm_bound = ws_mb > 100 and intensity < balance
    hbm_ach = kern_bytes / (kern_ms[k_dom] * 1e-3) / 1e9
    if hbm_bound:
        head = {"bound": "hbm", "achieved": round(hbm_ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(hbm_ach / hbm_peak, 4),
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "bytes_per_launch": kern_bytes,
                "bytes_rule": ("DRAM bytes this one-sweep kernel must move (Z stays on chip): "
                               + ("Y + B in, R out" if k_dom == 0 else "R + Y + X_prev in, X and Y out"))
                              if fused[k_dom >> 1] else
                              "DRAM bytes this kernel must move in the two-sweep design: "
                              + ("X in, r Z^T planes out" if k_dom in (0, 2) else
                                 "r Z^T planes + B in, R out" if k_dom == 1 else "r Z^T planes + Y + X_prev in, X and Y out"),
                "tensor": {"achieved": round(achieved_tf, 3), "peak": round(peak_dom, 3), "unit": "TFLOP/s",
                           "frac": round(achieved_tf / peak_dom, 4), "peak_source": peak_src}}
    else:
        head = {"bound": "tensor", "achieved": round(achieved_tf, 3), "peak": round(peak_dom, 3), "unit": "TFLOP/s",
                "frac": round(achieved_tf / peak_dom, 4),
                "peak_source": "measured live by kb_fma_peak in this run: " + peak_src}
    res["roofline"] = {
        **head,
        "kernel": f"{phase[k_dom]} on {engines[k_dom]}: the longest of the iteration's kernels",
        "intensity_flop_per_byte": round(intensity, 2), "machine_balance_flop_per_byte": round(balance, 2),
        "flops_per_launch": flops_phase[k_dom],
        "flops_rule": f"2 r w_exec flop per pixel and pass: r={cfg.r}, executed taps {wa} (axis 0) / {wb} (axis 1)"
                      + ("; axis-swapped twin: pass A = axis 1" if swapped else "")
                      + ("; a fused launch runs both passes of its direction" if fused[k_dom >> 1] else ""),
        "traffic": traffic[k_dom] if traffic else None,
        "traffic_source": f"profiles/traffic_{cfg.name}.json (ncu --set full, dram read+write of this kernel)",
        "kernel_dram_bytes_compulsory": kern_bytes,
        "kernel_hbm_frac": round(hbm_ach / hbm_peak, 4),
        "iteration": {
            "per_kernel_ms": [round(x, 5) for x in kern_ms],
            "engines": engines,
            "achieved_tflops": round(sum(flops_phase) / (it_ms * 1e-3) / 1e12, 3),
            "frac_of_peak": [round(f / (t * 1e-3) / 1e12 / engine_peak(e)[0], 4) if t > 0 else None
                             for f, t, e in zip(flops_phase, kern_ms, engines)],
        },
        "hbm": {"achieved": round(8 * esz * px / (it_ms * 1e-3) / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(8 * esz * px / (it_ms * 1e-3) / 1e9 / hbm_peak, 4), "peak_source": peak_kind,
                "algorithmic_bytes_per_px_it": 8 * esz,
                "note": "SURVEY 8(d) two-sweep compulsory bytes (Z planes excluded) over the iteration's kernels"},
        "nominal_flops_per_px_it": algorithmic(cfg),
        "executed_taps": [wa, wb],
    }
    if traffic and len(traffic) == 4 and all(t >= 0 for t in traffic):
        # the whole iteration's DRAM bytes as ncu measured them (committed capture of the same
        # kernels) over this run's iteration time: how close the iteration runs to the HBM roof
        tb = float(sum(traffic))
        res["roofline"]["iteration"]["dram_bytes_ncu"] = int(tb)
        res["roofline"]["iteration"]["dram_frac"] = round(tb / (it_ms * 1e-3) / 1e9 / hbm_peak, 4)
    if engines_solve and engines_solve[0] == "persist_f64":
        # one cooperative launch runs the whole solve: its roofline is the solve's own rate
        per_it_s = ms * 1e-3 / iters
        ach = sum(flops_phase) / per_it_s / 1e12
        pk, src = engine_peak("dmma")
        # kb_capi.cu persist2_plan: zero BC, half widths <= 15, r <= 4, n % 64 == 0, n <= 512
        second = (dev.bc == (0, 0) and max(dev.half_widths) <= 15 and cfg.r <= 4 and m % 64 == 0 and m <= 512
                  and os.environ.get("KB_PERSIST2", "1") != "0")
        res["roofline"].update({
            "bound": "tensor", "unit": "TFLOP/s",
            "kernel": ("kb_solve_persistent2" if second else "kb_solve_persistent")
                      + " (whole solve in one cooperative launch, 2 grid barriers per iteration)",
            "achieved": round(ach, 3), "peak": round(pk, 3), "frac": round(ach / pk, 4),
            "flops_per_launch": sum(flops_phase) * iters,
            "peak_source": "measured live by kb_fma_peak in this run: " + src + " (FP64 FMA has the same nominal rate)"})
    res["dev"] = dev
    del Bd, Xd, Yd, flush
    return res


def run_b200(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1901_00913_b200 import workloads as W

    cfg = W.CONFIGS[args.config]
    dtype = args.dtype or default_dtype(cfg)

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

    res = measure_config(args.config, dtype, args.steps, args.warmup, rank, world, local, clocks=True,
                         e2e_steps=max(3, min(args.steps, 10)), barrier=barrier, max_over_ranks=max_over_ranks)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample_line(cfg, res["op"] if not res["batched"] else res["ops"][0], samples=3)
    variants = {}
    if not args.no_variants and world == 1:
        for vname, vdt in VARIANTS:
            if (vname, vdt) == (args.config, dtype):
                continue
            res_keep = res.pop("dev", None)
            del res_keep
            torch.cuda.empty_cache()
            v = measure_config(vname, vdt, 3, 3, rank, world, local, e2e_steps=2)
            variants[f"{vname}_{vdt}"] = {
                "value": round(v["value"], 2), "ms_per_step": round(v["ms"], 4),
                "e2e": round(v["e2e"]["value"], 2), "engines": v["engines_solve"],
                "roofline_frac": v["roofline"]["frac"], "kernel": v["roofline"]["kernel"],
                "per_kernel_ms": v["roofline"]["iteration"]["per_kernel_ms"],
                "workload": workload_name(v["cfg"], v["batched"]),
            }
            del v
            torch.cuda.empty_cache()
    if rank == 0:
        line = {
            "metric": "sFISTA Mpixel*iterations/s",
            "value": round(res["value"], 2),
            "unit": "Mpixel*iterations/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(res["ms"], 4),
            "higher_is_better": True,
            "scaling": "strong" if res["batched"] else "weak",
            "vs_baseline": None,
            "dtype": "f64" if dtype == "float64" else "f32",
            "data": f"synthetic (seeded phantom + PSF + exact-level Gaussian noise, BASELINE {cfg.name})",
            "config": config_dict(cfg, dtype, world),
            "e2e": res["e2e"],
            "roofline": res["roofline"],
            "gpu_launches": res["launches"],
            "engines": res["engines_solve"],
            "clocks": res["clocks"],
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


def config_dict(cfg, dtype, world):
    """The `config` object of a line (identical for the b200 and reference arms of a config)."""
    batched = cfg.batch > 1
    return {"workload": workload_name(cfg, batched),
            "global_batch": cfg.batch if batched else world,
            "parallelism": f"batch-shard{world}" if batched else f"replicas{world}",
            "l2": l2_note(cfg, dtype, cfg.batch)}


def workload_name(cfg, batched):
    return (f"{cfg.name}: {(str(cfg.batch) + ' x ') if batched else ''}{cfg.m}x{cfg.m} {cfg.bc} BC, "
            f"w={cfg.w}, r={cfg.r}, lam={cfg.lam}, x>=0, {cfg.iters} iterations per step")


def run_row_blocks(args):
    """cfg4 / cfg5 at N > 1 (or --row-blocks at N = 1): ONE image split into contiguous row blocks
    across ranks, shard.solve_row_blocks with two halo exchanges per iteration over
    NCCL (batch_isend_irecv). Strong scaling: value = m*m*iters of the whole image / max-over-ranks
    solve time. Every rank generates the same seeded image (setup: the Philox noise stream is
    drawn whole) and keeps its rows; L comes from the sharded power iteration (halo exchanges,
    <v, w> and ||w||^2 all-reduced, shard.power_iter_row_blocks) in fp64."""
    import torch

    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200 import workloads as W
    from paper_1901_00913_b200.device import fma_peak
    from paper_1901_00913_b200.shard import (BlockPlan, DeviceBlockBackend, halo_rows, power_iter_row_blocks,
                                             prefer_swap, solve_row_blocks, swapped)
    from paper_1901_00913_b200.solvers import _start_vector

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.CONFIGS[args.config]
    args.dtype = args.dtype or default_dtype(cfg)
    m, iters = cfg.m, cfg.iters
    B, op, _ = build_problem(cfg, args.dtype, seed=0, lipschitz=False)
    # the single-GPU fast path's axis swap (wider band in pass A): shard the transposed image
    swap = prefer_swap(op, args.dtype)
    if swap:
        op, B = swapped(op), np.ascontiguousarray(B.T)
    plan = BlockPlan(m, m, world, rank, halo_rows(op))
    # L: matrix-form power iteration (50 steps, fp64, seed 0) sharded like the solve (transposed
    # start vector in the swapped frame: the same sequence)
    back64 = DeviceBlockBackend(op, plan, "float64")
    v0 = _start_vector(0, m, m, "matrix")
    v0 = (v0.T if swap else v0)[plan.g0:plan.g0 + plan.rows]
    L = power_iter_row_blocks(back64, plan, torch.from_numpy(np.ascontiguousarray(v0)).cuda(), 50)
    del back64
    torch.cuda.empty_cache()
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
    wa, wb = backend.dev.bands[1], backend.dev.bands[3]  # executed taps
    achieved = 4 * cfg.r * (wa + wb) * m * m * iters / (ms * 1e-3) / 1e12 / world  # per GPU
    overlap = plan.overlap_ranges() is not None
    launches = (12 if overlap else 4) * iters * args.steps
    if rank == 0:
        line = {
            "metric": "sFISTA Mpixel*iterations/s", "value": round(value, 2), "unit": "Mpixel*iterations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.dtype == "float64" else "f32",
            "data": f"synthetic (seeded phantom + PSF + exact-level Gaussian noise, BASELINE {cfg.name})",
            "config": {"workload": f"{args.config}: {m}x{m} {cfg.bc} BC, w={cfg.w}, r={cfg.r}, lam={cfg.lam}, "
                                   f"x>=0, {iters} iterations per step, row blocks of {plan.rows} rows, "
                                   f"halo {plan.h}" + (", interior/halo overlap" if overlap else "")
                                   + (", transposed image (axis swap)" if swap else ""),
                       "global_batch": 1, "parallelism": f"row-blocks{world}",
                       "l2": "flushed between steps (256 MiB write); HBM-backed working set"},
            "e2e": {"value": m * m * iters / 1e6 / e2e_s, "unit": "Mpixel*iterations/s",
                    "h2d_bytes_per_step": m * m * esz, "d2h_bytes_per_step": m * m * esz},
            "roofline": {"bound": "tensor", "kernel": f"whole row-block iteration per GPU ({eng} passes, "
                                                      "halo exchanges included)",
                         "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "flops_rule": f"4 r (w_a + w_b) per pixel-iteration, executed taps {wa}/{wb}"},
            "lipschitz": L,
            "gpu_launches": launches,
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


def cpu_sample(cfg, op, threads, B=None, L=1.0, cols=2048):
    """One bounded sample of the reference's CPU hot path (oracle port = kronblur's numpy
    pocketfft path, solvers.py:168-176 / structured.py:184-198) on this config, extrapolated to
    one sFISTA iteration. Returns (seconds per iteration, sample description, sample seconds).

    m <= 2048: one whole projected iteration (kron_apply + kron_apply_adjoint + update).
    Larger: one factor application (term 1's H, order m, Toeplitz(+Hankel) FFT apply) to an
    m x `cols` column block; an iteration is 4 r such applications over all n columns (forward
    H_i and K_i, adjoint H_i^T and K_i^T per term), i.e. 4 r n / cols samples. The elementwise
    update (~1-2 % at 1024^2) is not extrapolated."""
    from oracle import kronblur_port as port

    port.set_threads(threads)
    m, n = op.shape
    if m <= 2048:
        pop = port.PortOperator(op)
        Bh = B if B is not None else np.random.default_rng(0).random((m, n))
        t0 = time.perf_counter()
        port.sfista(pop, Bh, L, cfg.lam, 1, project=True)
        dt = time.perf_counter() - t0
        return dt, f"one projected sFISTA iteration of {cfg.name} ({m}x{n}, fp64, numpy pocketfft path)", dt
    cols = min(cols, n)
    plan = port.FactorPlan(op.terms[0].H)
    Xs = np.random.default_rng(0).random((m, cols))
    port.factor_apply(plan, Xs[:, :64])  # warm the FFT plan caches
    t0 = time.perf_counter()
    port.factor_apply(plan, Xs)
    dt = time.perf_counter() - t0
    per_iter = dt * 4 * cfg.r * (n / cols)
    return per_iter, (f"one Toeplitz+Hankel factor application (order {m}, numpy pocketfft path) to a {m}x{cols} "
                      f"column block of {cfg.name}, x 4r n/cols = {4 * cfg.r * n // cols} to one iteration"), dt


def cpu_sample_line(cfg, op, samples=3, threads=None, B=None, L=1.0):
    threads = threads or cpu_threads()
    best = None
    for _ in range(samples):
        per_iter, what, dt = cpu_sample(cfg, op, threads, B, L)
        best = per_iter if best is None else min(best, per_iter)
    value = cfg.batch * cfg.m * cfg.m / best / 1e6 if cfg.batch == 1 else cfg.m * cfg.m / best / 1e6
    return {"value": round(value, 4), "unit": "Mpixel*iterations/s", "cores": threads, "kind": "port",
            "sample": f"{what}; best of {samples} samples ({dt:.2f} s each)", "same_config": True}


def run_reference(args):
    """The reference arm: kronblur's CPU hot path (the oracle port) on this box's host cores, on
    the same config, metric and unit as the b200 arm; each step is one bounded sample of an
    iteration (cpu_sample), so `--steps K --warmup W` ends within minutes even at cfg5."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200 import workloads as W

    cfg = W.CONFIGS[args.config]
    psf = W.make_psf(cfg, index=0, seed=0)
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
    threads = cpu_threads()
    B = None
    if cfg.m <= 2048:  # small configs: the real data (CPU blur by the numpy port)
        from oracle import kronblur_port as port

        X = W.phantom(cfg.m, cfg.n_rect, cfg.n_disk, 0, device="cpu").numpy()
        B = W.add_noise(port.blur_direct(psf.values, psf.center, X, cfg.bc), cfg.noise, 0)
    times, walls, what = [], [], ""
    for s in range(args.warmup + args.steps):
        per_iter, what, wall = cpu_sample(cfg, op, threads, B, 1.0)
        if s >= args.warmup:
            times.append(per_iter)
            walls.append(wall)
    step = sum(times) / len(times)
    value = cfg.m * cfg.m / step / 1e6  # per image; cfg3's batch is independent images
    line = {
        "metric": "sFISTA Mpixel*iterations/s", "value": round(value, 4), "unit": "Mpixel*iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sum(walls) / len(walls) * 1e3, 3),  # wall time of one sample (one step)
        "ms_per_iteration_extrapolated": round(step * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {cfg.name})",
        "config": config_dict(cfg, default_dtype(cfg), 1),
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpixel*iterations/s", "cores": threads,
                         "kind": "port", "sample": what, "same_config": True},
        "e2e": {"value": round(value, 4), "unit": "Mpixel*iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: re-execute under torch.distributed.run with N
    ranks on this node (rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port_no = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port_no), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    rank, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.config in ("cfg4", "cfg5") and (args.row_blocks or world > 1):
        run_row_blocks(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

"""Benchmark of the B200 batched piecewise sin/cos/tan path (arXiv 2502.10831).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--configs auto|none|cfg1,cfg3,...] [--elements N]
                    [--backend nccl|gloo] [--f32-policy ulp2|bitwise]
                    [--no-e2e] [--no-cpu] [--e2e-elements N] [--e2e-steps S]

Headline (N=1): BASELINE.json configs[1] -- f64 x, 2^28 elements uniform in
[-1000pi, 1000pi], fused proposed sin+cos+tan (three output arrays), default
SqrtMode (fisr, 1 Newton step).  Under torchrun each rank owns a contiguous
2^28-element shard of one global array (global index = generator counter):
per-GPU work is fixed, so "scaling": "weak".  No element data moves between
GPUs; after each timed region every rank runs the K3 parity/error reduction and
the ranks all-reduce the 312-byte statistics (max / sum), the only collective.

The same run also times every other BASELINE config and reports it under
`configs` (value, ms, roofline, FP64 roof, clocks, K3 accuracy each): cfg1, cfg3,
cfg4_f32, cfg4_f64 weak-scaled per GPU, and cfg5 -- the fixed 2^33-element f32
array -- strong-scaled (N=1: all 2^33 elements on one GPU; N>1: 2^33/N each).

One step = one K1/K2 launch sequence over the shard (inputs already resident in
HBM).  L2: the headline's x + outputs are 8 GiB per GPU (>> 126 MB L2), no
flush; configs whose input is smaller than L2 (cfg1: 64 MiB) rotate the timed
steps over identical copies of the batch in distinct buffers, so that >= 2x L2
of other traffic separates two reads of one x (every step reads x from HBM,
with no flush kernel and its dirty-line write-back inside the timing).  Timing: CUDA
events on the launching stream, barrier + synchronize on both sides, max over
ranks.

`sustained` repeats the headline step for ~20 s of device time (the
power-capped steady state; the headline window is under a second).  `burst`
(headline and every config) is the best of 3 windows of ~20 ms of back-to-back
steps, each after 1 s of idle and ~5 ms of untimed launches: the rate before
the board-power limiter engages (~50 ms into a run, tools/power_ramp.py), i.e.
the regime the HBM peak itself (best of 10 single copies) is measured in.

`e2e` is the headline metric through the public host-pointer C-ABI call
(ft_proposed_batch_host) with pinned host buffers over the full shard: every
step copies x in and sin/cos/tan out.  `e2e_variants` adds the reference-shaped
seams: the three single-output calls ft_proposed_{sin,cos,tan}_batch on
pageable (malloc'd) buffers -- what fasttrig::gpu::proposed_*_batch with
std::vector does -- and the fused call on pageable buffers.  `cpu_baseline`
(rank 0, N=1) and `--impl reference` time the reference's own CPU
implementation (oracle/_ref: the unmodified reference headers, all host
threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gelem/s per GPU and box (1/2/4/8 B200); % of HBM/FP64 roofline; max abs err"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


def env_int(k: str, d: int) -> int:
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_summary() -> dict:
    """The committed ncu --set full summary of K1/K2 (profiles/ncu_k1_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_k1_summary.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic(workload: str):
    """Per-launch DRAM bytes of K1 from the committed ncu --set full summary, if any."""
    return ncu_summary().get("traffic_bytes_per_launch", {}).get(workload)


def fp64_roof(workload: str, gelem_s_per_gpu: float):
    """The FP64-pipe roof beside the HBM one: issued FP64-pipe instructions per
    element (ncu, this kernel) x throughput vs the measured DFMA lane-op peak."""
    d = ncu_summary()
    ops = d.get("fp64_pipe_instr_per_elem", {}).get(workload)
    peak = d.get("fp64_peak_lane_ops_per_s")
    if not ops or not peak:
        return None
    ach = ops * gelem_s_per_gpu * 1e9
    return {"bound": "fp64", "ops_per_elem": ops, "achieved": round(ach / 1e12, 3),
            "peak": round(peak / 1e12, 3), "unit": "T lane-ops/s", "frac": round(ach / peak, 4),
            "source": "ops/elem from profiles/ncu_k1_summary.json; peak " + d.get("fp64_peak_source", "")}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,clocks.mem")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def mark(self):
        """Samples taken before the last mark() are dropped (idle / setup)."""
        self.t_mark = time.time()

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        self.t_mark = 0.0
        time.sleep(0.2)  # let nvidia-smi start sampling

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        import datetime

        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if ts < self.t_mark:
                    continue
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
            try:
                pw.append(float(parts[8]))
            except (ValueError, IndexError):
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "samples": len(sm),
                "reasons": sorted(reasons),
                "power_w_median": statistics.median(pw) if pw else None}


# ------------------------------------------------------------------ CPU baseline
def cpu_rate(get_x, mask: int, threads: int, target_s: float, kind_pref: str = "reference"):
    """Time the reference CPU path (oracle/_ref) -- or the C port when the reference
    was not built -- on get_x(n) (a prefix of the workload's own input stream, n sized
    to take ~target_s).  Returns (gelem_per_s, kind, n_sample, seconds, x_sample)."""
    from oracle import oracle as O

    kind = "reference" if (kind_pref == "reference" and O.ref_available()) else "port"
    impl = "ref" if kind == "reference" else "port"
    probe = get_x(1 << 18)
    O.proposed(probe, mask, threads=threads, impl=impl)  # warm
    t0 = time.perf_counter()
    O.proposed(probe, mask, threads=threads, impl=impl)
    dt = max(time.perf_counter() - t0, 1e-6)
    n = int(min(1 << 28, max(1 << 18, probe.size * target_s / dt)))
    x = get_x(n)
    t0 = time.perf_counter()
    O.proposed(x, mask, threads=threads, impl=impl)
    dt = time.perf_counter() - t0
    return x.size / dt / 1e9, kind, x.size, dt, x


def api_single_thread_rate(w, n: int = 1 << 20):
    """The reference's own batch API, exactly as a caller uses it (R:kernels.hpp:84-94:
    one thread, allocates a std::vector per call), for sin, cos and tan in turn.
    Returns Gelem/s of fused-equivalent work (elements / total time of the 3 calls)."""
    import numpy as np

    from oracle import oracle as O

    if not O.ref_available():
        return None
    x = O.gen_uniform(n, w.lo, w.hi, w.seed, 0, np.float64)
    out = np.empty_like(x)
    R = O.ref()
    best = float("inf")
    for _ in range(3):
        t0 = time.perf_counter()
        for which in range(3):
            R.ref_api_batch(which, x.ctypes.data, n, 1, 1, out.ctypes.data)
        best = min(best, time.perf_counter() - t0)
    return n / best / 1e9


def host_inputs(w):
    """Host copy of the first n elements of workload w's input stream (uniform
    configs are generated on the host bit-identically to K4)."""
    import numpy as np

    from oracle import oracle as O

    def get(n: int):
        return O.gen_uniform(n, w.lo, w.hi, w.seed, 0, np.dtype(w.dtype).type)
    return get


def host_cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------ shared
# Timed steps per extra config (~0.2-1 s of timed work each at N=1).
CONFIG_STEPS = {"cfg1": 2000, "cfg2": 600, "cfg3": 1000, "cfg4_f32": 400, "cfg4_f64": 300, "cfg5": 20}
EXTRA_CONFIGS = ("cfg1", "cfg3", "cfg4_f32", "cfg4_f64", "cfg5")
L2_BYTES = 126 * 1000 * 1000


def plan(w, world: int, rank: int, elements: int = 0):
    """(n on this rank, global offset, scaling, total elements) for workload w.
    cfg5 is one fixed global array split over the ranks (strong); the others give
    every rank its own shard of w.n (or `elements`) elements (weak)."""
    from paper_2502_10831_b200.configs import shard

    if w.name == "cfg5":
        total = elements or w.n
        lo, hi = shard(total, rank, world)
        return hi - lo, lo, "strong", total
    n = elements or w.n
    return n, rank * n, "weak", n * world


def config_dict(w, n: int, world: int, policy: str, rotate: int) -> dict:
    """The `config` object of a line: identical for our arm and the reference arm."""
    names = [nm for j, nm in enumerate(("sin", "cos", "tan")) if w.mask & (1 << j)]
    step_bytes = w.bytes_per_elem * n
    d = {"workload": w.name, "description": w.note, "elements_per_gpu": n, "outputs": names,
         "sqrt_mode": "fisr(1) (SqrtMode{} default)" if w.kind == 0 else f"Taylor-{w.n_terms}",
         "parallelism": f"dp{world} contiguous shards, no data exchange",
         "l2": (f"x ({w.itemsize * n / 2**20:.0f} MiB) smaller than L2: timed steps rotate over {rotate} "
                f"copies of the batch (x + outputs = {rotate * step_bytes / 2**20:.0f} MiB, "
                f"{rotate * step_bytes / L2_BYTES:.1f}x L2), so every step reads its x from HBM; no flush"
                if rotate > 1 else f"inputs larger than L2 (x + outputs = {step_bytes / 2**30:.1f} GiB "
                                   "per GPU vs 126 MB L2); no flush")}
    if w.itemsize == 4:
        d["f32_policy"] = policy
    return d


def rotation(w, n: int) -> int:
    """Buffer sets the timed steps cycle through: 1 when x alone exceeds L2, else
    enough copies that the other sets' traffic between two uses of one set is
    >= 2x L2 (x is then evicted before it is read again)."""
    if w.itemsize * n >= L2_BYTES:
        return 1
    step = w.bytes_per_elem * n
    return 1 + max(2, -(-2 * L2_BYTES // step))


# ------------------------------------------------------------------ reference arm
def reference_sample(steps: int, warmup: int) -> int:
    """Elements per reference step: the whole 2^28 headline shard when the run is
    short, else a power-of-two slice so that (steps + warmup) steps stay within
    a few minutes; deterministic (does not depend on the host's speed)."""
    n = 1 << 28
    total = max(1, steps + warmup)
    while n > (1 << 20) and n * total > (1 << 28) * 64:
        n >>= 1
    return n


def run_reference(args) -> None:
    rank = env_int("RANK", 0)
    if rank != 0:
        return  # the reference arm is single-process CPU work; other ranks idle
    from oracle import oracle as O
    from paper_2502_10831_b200.configs import CONFIGS

    w = CONFIGS[args.config]
    threads = O.ncpu()
    n_cfg, _, scaling, _ = plan(w, 1, 0, args.elements)
    n = min(n_cfg, reference_sample(args.steps, args.warmup))
    kind = "reference" if O.ref_available() else "port"
    impl = "ref" if kind == "reference" else "port"
    x = host_inputs(w)(n)
    for _ in range(args.warmup):
        O.proposed(x, w.mask, threads=threads, impl=impl)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.proposed(x, w.mask, threads=threads, impl=impl)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    value = n / (ms / 1e3) / 1e9
    sample = (f"first {n} elements of {w.name} per step ({w.note}); fused sin+cos+tan via the scalar "
              f"reference calls, contiguous partition over {threads} threads; {host_cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gelem/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64" if w.itemsize == 8 else "f32", "data": "synthetic",
        "config": config_dict(w, n_cfg, args.gpus, args.f32_policy, rotation(w, n_cfg)),
        "cpu_baseline": {"value": round(value, 6), "unit": "Gelem/s", "cores": threads,
                         "kind": kind, "sample": sample, "elements_per_step": n,
                         "api_batch_single_thread_gelem_s": api_single_thread_rate(w)},
        "e2e": {"value": round(value, 6), "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
class Ctx:
    """Per-process state of our arm: rank layout, device, collectives."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.args = args
        self.world = env_int("WORLD_SIZE", 1)
        self.rank = env_int("RANK", 0)
        local = env_int("LOCAL_RANK", 0)
        if self.world != args.gpus and self.world > 1:
            print(f"warning: WORLD_SIZE={self.world} but --gpus {args.gpus}", file=sys.stderr)
        ndev = torch.cuda.device_count()
        self.device_index = local % max(1, ndev)  # gloo test runs put several ranks on one GPU
        torch.cuda.set_device(self.device_index)
        self.dev = torch.device("cuda", self.device_index)
        launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # torchrun
        self.backend = args.backend
        if self.world > 1 or launched:
            if self.backend == "nccl":
                # communicator INIT lines (rank count, NVLS / ring setup) into the log
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")
        self.dist = dist

    @property
    def coll_device(self):
        return self.dev if self.backend == "nccl" else "cpu"

    def barrier(self):
        if self.dist.is_initialized():
            self.dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        import torch

        t = torch.tensor([v], dtype=torch.float64, device=self.coll_device)
        if self.dist.is_initialized() and self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def time_steps(step, k: int, stream) -> float:
    """Mean device time of one step (ms) over k back-to-back steps, CUDA events
    on `stream`; step(i) runs the i-th step."""
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(k):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def burst_window(ctx: Ctx, step, stream, ms_hint: float, window_ms: float = 20.0, idle_s: float = 1.0,
                 reps: int = 3) -> dict:
    """Best of `reps` short windows (~`window_ms` of back-to-back steps, >= 3),
    each after `idle_s` of idle and ~5 ms of untimed launches: the rate before
    the board-power limiter engages (it does ~50 ms into a run of the f32
    kernels, tools/power_ramp.py) -- the regime MEASURED_PEAKS.json's hbm_gbs
    (best of 10 single copies) is measured in."""
    import torch

    k = max(3, int(window_ms / max(ms_hint, 1e-3)))
    kw = max(3, int(5.0 / max(ms_hint, 1e-3)))
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        time.sleep(idle_s)
        ctx.barrier()
        for i in range(kw):
            step(i)
        best = min(best, ctx.max_over_ranks(time_steps(step, k, stream)))
    return {"ms_per_step": best, "steps": k, "warmup": kw, "idle_s": idle_s, "reps": reps}


def measure(ctx: Ctx, w, steps: int, warmup: int, policy: str, elements: int = 0, keep: bool = False,
            burst: bool = True):
    """Generate w's shard in place, time `steps` launches of its kernel, check
    the outputs with K3, all-reduce the statistics.  Returns (entry, state)."""
    import torch

    import paper_2502_10831_b200 as ft
    from paper_2502_10831_b200.dist import reduce_stats

    n, lo, scaling, total = plan(w, ctx.world, ctx.rank, elements)
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    x = torch.empty(n, dtype=tdt, device="cuda")
    ft.gen_inputs(min(n, 1 << 16), tdt, w.dist, w.lo, w.hi, w.seed, lo, out=x)  # module load outside the timing
    torch.cuda.synchronize()
    ev[0].record(stream)
    ft.gen_inputs(n, tdt, w.dist, w.lo, w.hi, w.seed, lo, out=x)  # K4: generated in place, global index as the counter
    ev[1].record(stream)
    names = [nm for j, nm in enumerate(("sin", "cos", "tan")) if w.mask & (1 << j)]
    out = {nm: torch.empty_like(x) for nm in names}
    mode = ft.SqrtMode()
    rot = rotation(w, n)
    # identical copies of the batch in distinct buffers (see rotation())
    sets = [(x, out)] + [(x.clone(), {nm: torch.empty_like(x) for nm in names}) for _ in range(rot - 1)]

    def step(i=0):
        xi, oi = sets[i % rot]
        if w.kind == 0:
            ft.proposed_eval(xi, w.mask, mode, out=oi)
        else:
            ft.taylor_eval(xi, w.n_terms, w.mask, out=oi)

    with ft.f32_policy(policy):
        clocks = ClockSampler(ctx.device_index)  # samples from warm-up start to timed-region end
        clocks.start()
        clocks.mark()
        for _ in range(max(warmup, 3)):
            step()
        torch.cuda.synchronize()
        ctx.barrier()
        torch.cuda.synchronize()
        l0 = ft.launch_count()
        ms_local = time_steps(step, steps, stream)
        ctx.barrier()
        launches = ft.launch_count() - l0
        clk = clocks.stop()
        bw = burst_window(ctx, step, stream, ms_local) if burst else None
        # cfg5 at N=1: one step (2^33 elements, 8 chained launches) is longer than
        # the pre-limiter window, so also time the shard each GPU of the 8-GPU
        # configuration processes (2^30 elements, one launch) in that window
        bshard = None
        if burst and w.name == "cfg5" and ctx.world == 1 and n > (1 << 30):
            ns = 1 << 30
            xs_, os_ = x[:ns], {nm: o[:ns] for nm, o in out.items()}

            def step_shard(i=0):
                ft.proposed_eval(xs_, w.mask, mode, out=os_)

            bshard = burst_window(ctx, step_shard, stream, ms_local * ns / n)
            bshard["elements"] = ns
    ms = ctx.max_over_ranks(ms_local)
    value = total / (ms / 1e3) / 1e9

    peak, peak_src = peaks()
    achieved = w.bytes_per_elem * n / (ms_local / 1e3) / 1e9
    traffic = ncu_traffic(w.name)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed "
                                   "ncu --set full capture (profiles/ncu_k1_summary.json; static, not measured "
                                   "in this run)") if traffic else None,
                "peak_source": peak_src, "algorithmic_bytes_per_elem": w.bytes_per_elem,
                "kernel": ("k_proposed (K1)" if w.kind == 0 else "k_taylor (K2)")
                + (" relaxed f32" if w.itemsize == 4 and policy == "ulp2" else "")}

    m_warm = min(n, 1 << 16)  # K3's module load outside its timing
    ft.parity_reduce(x[:m_warm], {nm: o[:m_warm] for nm, o in out.items()}, w.mask, kind=w.kind, mode=mode,
                     n_terms=w.n_terms, ulp_tol=2)
    ev[2].record(stream)
    st = ft.parity_reduce(x, out, w.mask, kind=w.kind, mode=mode, n_terms=w.n_terms, ulp_tol=2)
    ev[3].record(stream)
    torch.cuda.synchronize()
    k4_ms, k3_ms = ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])
    # the path's other two kernels, one launch sequence each, outside the timed region (this rank's shard)
    aux = {"k4_gen_inputs": {"gelem_s": round(n / (k4_ms / 1e3) / 1e9, 2), "ms": round(k4_ms, 3),
                             "gbs_written": round(n * w.itemsize / (k4_ms / 1e3) / 1e9, 1)},
           "k3_parity_reduce": {"gelem_s": round(n / (k3_ms / 1e3) / 1e9, 2), "ms": round(k3_ms, 3),
                                "note": "per element: the device restatement of every requested function "
                                        "(IEEE divisions) + CUDA libm sin/cos/tan in binary64; FP64-pipe bound"}}
    st = reduce_stats(st, device=ctx.coll_device)  # the path's only collective: 312 B of stats
    accuracy = {
        "checked": int(st["n_checked"]), "max_ulp_vs_oracle": st["max_ulp"], "tolerance_ulp": 2,
        "over_2ulp": st["n_over_tol"], "bit_mismatch_vs_oracle": st["n_bit_mismatch"],
        "max_abs_err_vs_libm": st["max_abs_vs_libm"], "max_rel_err_vs_libm": st["max_rel_vs_libm"],
        "avg_abs_err_vs_libm": [s_ / max(1, c) for s_, c in zip(st["sum_abs_vs_libm"], st["n_finite_libm"])],
        "max_abs_err_vs_oracle": st["max_abs_vs_oracle"], "inf_count": st["n_inf"],
        "nan_count": st["n_nan"], "checksum": st["checksum"], "outputs": names,
        "oracle": "device restatement of the reference (ft_mirror_*), bitwise-pinned to the CPU oracle",
    }
    # configs[3]: "measured side by side with the piecewise kernel" -- the proposed
    # functions of the same mask on the same x, same steps, same checks
    side = None
    if w.kind == 1:
        out_p = {nm: torch.empty_like(x) for nm in names}

        def step_p(i=0):
            ft.proposed_eval(x, w.mask, mode, out=out_p)

        with ft.f32_policy(policy):
            for _ in range(3):
                step_p()
            torch.cuda.synchronize()
            ctx.barrier()
            ms_p_local = time_steps(step_p, steps, stream)
            ctx.barrier()
        ms_p = ctx.max_over_ranks(ms_p_local)
        st_p = reduce_stats(ft.parity_reduce(x, out_p, w.mask, kind=0, mode=mode, ulp_tol=2), device=ctx.coll_device)
        side = {"kernel": "k_proposed (K1)" + (" relaxed f32" if w.itemsize == 4 and policy == "ulp2" else ""),
                "outputs": names, "value": round(total / (ms_p / 1e3) / 1e9, 4), "unit": "Gelem/s",
                "ms_per_step": round(ms_p, 5), "steps": steps,
                "roofline_frac": round(w.bytes_per_elem * n / (ms_p_local / 1e3) / 1e9 / peak, 4),
                "max_ulp_vs_oracle": st_p["max_ulp"], "max_abs_err_vs_libm": st_p["max_abs_vs_libm"],
                "avg_abs_err_vs_libm": [s_ / max(1, c) for s_, c in zip(st_p["sum_abs_vs_libm"],
                                                                         st_p["n_finite_libm"])]}
        del out_p
    if bw:
        bms = bw["ms_per_step"]
        bw = {"value": round(total / (bms / 1e3) / 1e9, 4), "unit": "Gelem/s", "ms_per_step": round(bms, 5),
              "steps": bw["steps"], "warmup": bw["warmup"], "idle_s": bw["idle_s"], "best_of": bw["reps"],
              "roofline_frac": round(w.bytes_per_elem * n / (bms / 1e3) / 1e9 / peak, 4)}
    entry = {"value": round(value, 4), "unit": "Gelem/s", "per_gpu_gelem_s": round(n / (ms / 1e3) / 1e9, 4),
             "ms_per_step": round(ms, 5), "steps": steps, "warmup": max(warmup, 3), "scaling": scaling,
             "dtype": "f64" if w.itemsize == 8 else "f32",
             "config": config_dict(w, n, ctx.world, policy, rot), "roofline": roofline,
             "fp64_roof": fp64_roof(w.name, n / (ms_local / 1e3) / 1e9), "gpu_launches": int(launches),
             "clocks": clk, "burst": bw, "aux_kernels": aux, "accuracy": accuracy}
    if bshard:
        sms = bshard["ms_per_step"]
        entry["burst_8gpu_shard"] = {
            "elements": bshard["elements"], "value": round(bshard["elements"] / (sms / 1e3) / 1e9, 4),
            "unit": "Gelem/s", "ms_per_step": round(sms, 5), "steps": bshard["steps"],
            "roofline_frac": round(w.bytes_per_elem * bshard["elements"] / (sms / 1e3) / 1e9 / peak, 4),
            "note": "one GPU's share of the 8-GPU configuration (2^33 / 8), timed alone on this GPU"}
    if side:
        entry["piecewise_side_by_side"] = side
    state = {"x": x, "out": out, "n": n, "total": total, "names": names, "tdt": tdt} if keep else None
    del sets
    if not keep:
        del x, out
        torch.cuda.empty_cache()
    return entry, state


def sustained(ctx: Ctx, w, state, seconds: float, ms_hint: float, policy: str) -> dict:
    """The headline step repeated back to back for ~`seconds` of device time on
    the same buffers (the power-capped steady state a long production batch
    sees, next to the short headline window)."""
    import torch

    import paper_2502_10831_b200 as ft

    x, out = state["x"], state["out"]
    mode = ft.SqrtMode()
    k = max(10, int(seconds * 1e3 / max(ms_hint, 1e-3)))

    def step(i=0):
        if w.kind == 0:
            ft.proposed_eval(x, w.mask, mode, out=out)
        else:
            ft.taylor_eval(x, w.n_terms, w.mask, out=out)

    with ft.f32_policy(policy):
        clocks = ClockSampler(ctx.device_index)
        clocks.start()
        clocks.mark()
        torch.cuda.synchronize()
        ctx.barrier()
        ms_local = time_steps(step, k, torch.cuda.current_stream())
        ctx.barrier()
        clk = clocks.stop()
    ms = ctx.max_over_ranks(ms_local)
    n, total = state["n"], state["total"]
    peak, _ = peaks()
    return {"value": round(total / (ms / 1e3) / 1e9, 4), "unit": "Gelem/s", "ms_per_step": round(ms, 5),
            "steps": k, "seconds": round(k * ms / 1e3, 2),
            "roofline_frac": round(w.bytes_per_elem * n / (ms_local / 1e3) / 1e9 / peak, 4), "clocks": clk}


def e2e_pinned(ctx: Ctx, w, state, steps: int, n_e2e: int) -> dict:
    """The headline metric through the fused host-pointer C-ABI call, pinned
    host buffers, H2D of x and D2H of every output inside each timed step."""
    import torch

    from paper_2502_10831_b200 import _lib

    names, tdt = state["names"], state["tdt"]
    xh = torch.empty(n_e2e, dtype=tdt, pin_memory=True)
    xh.copy_(state["x"][:n_e2e])
    outs_h = {nm: torch.empty(n_e2e, dtype=tdt, pin_memory=True) for nm in names}
    ptr = [outs_h[nm].data_ptr() if nm in outs_h else None for nm in ("sin", "cos", "tan")]
    L = _lib.lib()
    dtc = _lib.FT_F32 if w.itemsize == 4 else _lib.FT_F64
    mode = _lib.SqrtModeC(1, 1)

    def call():
        if w.kind == 0:
            _lib.check(L.ft_proposed_batch_host(dtc, xh.data_ptr(), n_e2e, w.mask, mode, *ptr))
        else:
            _lib.check(L.ft_taylor_batch_host(dtc, xh.data_ptr(), n_e2e, w.mask, w.n_terms, *ptr))

    call()  # warm (allocates the pipeline buffers)
    ctx.barrier()
    times = []
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()  # blocking: returns with results in host memory
        times.append(time.perf_counter() - t0)
    t = ctx.max_over_ranks(statistics.mean(times))
    del xh, outs_h
    return {"value": round(n_e2e * ctx.world / t / 1e9, 6), "unit": "Gelem/s",
            "h2d_bytes_per_step": n_e2e * w.itemsize, "d2h_bytes_per_step": n_e2e * w.itemsize * len(names),
            "elements_per_step_per_gpu": n_e2e, "steps": steps,
            "timing": "host wall clock around the blocking fused C-ABI call (pinned buffers), max over ranks"}


def e2e_pageable(ctx: Ctx, w, state, steps: int, n_e2e: int) -> dict:
    """The reference-shaped seams on pageable host memory (numpy = malloc'd, as a
    std::vector is): (a) the three single-output calls ft_proposed_{sin,cos,tan}_batch
    per step -- what fasttrig::gpu::proposed_*_batch does --, (b) the fused call."""
    import numpy as np
    import torch

    from paper_2502_10831_b200 import _lib

    L = _lib.lib()
    mode = _lib.SqrtModeC(1, 1)
    res = {}
    if w.kind != 0 or w.itemsize != 8 or w.mask != 7:
        return res
    x = state["x"][:n_e2e].cpu().numpy()
    outs = {nm: np.empty_like(x) for nm in ("sin", "cos", "tan")}
    fns = (L.ft_proposed_sin_batch, L.ft_proposed_cos_batch, L.ft_proposed_tan_batch)

    def three():
        for f, nm in zip(fns, ("sin", "cos", "tan")):
            _lib.check(f(x.ctypes.data, n_e2e, mode, outs[nm].ctypes.data))

    def fused():
        _lib.check(L.ft_proposed_batch_host(_lib.FT_F64, x.ctypes.data, n_e2e, 7, mode,
                                            *[outs[nm].ctypes.data for nm in ("sin", "cos", "tan")]))

    # the C++ drop-in itself (gpu.hpp: std::vector in, a new std::vector out per call)
    exe = os.path.join(ROOT, "paper_2502_10831_b200", "lib", "bench_dropin")
    if ctx.world == 1 and os.path.exists(exe):
        try:
            r = subprocess.run([exe, str(n_e2e), str(steps)], capture_output=True, text=True, timeout=600)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            for key, val, note in (
                    ("cpp_gpu_hpp_x3_std_vector", d["api_x3_std_vector_gelem_s"],
                     "three calls, each returning a new std::vector"),
                    ("cpp_gpu_hpp_fused_std_vector", d["fused_std_vector_gelem_s"],
                     "proposed_sincostan_batch returning three new std::vectors"),
                    ("cpp_gpu_hpp_span_out", d["span_out_preallocated_gelem_s"],
                     "proposed_batch into caller-owned (pageable) vectors")):
                res[key] = {"value": round(val, 6), "unit": "Gelem/s", "elements_per_step_per_gpu": n_e2e,
                            "steps": steps, "call": note,
                            "new_std_vector_seconds": d["new_std_vector_seconds"],
                            "timing": "host steady_clock around the C++ calls (tools/bench_dropin.cpp)"}
        except Exception as e:  # noqa: BLE001 -- report, do not fail the bench line
            res["cpp_gpu_hpp_std_vector"] = {"error": repr(e)[:200]}
    for name, fn, h2d in (("api_single_output_x3_pageable", three, 3), ("fused_pageable", fused, 1)):
        fn()  # warm
        ctx.barrier()
        times = []
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            times.append(time.perf_counter() - t0)
        t = ctx.max_over_ranks(statistics.mean(times))
        res[name] = {"value": round(n_e2e * ctx.world / t / 1e9, 6), "unit": "Gelem/s",
                     "h2d_bytes_per_step": h2d * n_e2e * 8, "d2h_bytes_per_step": 3 * n_e2e * 8,
                     "elements_per_step_per_gpu": n_e2e, "steps": steps}
    return res


def run_ours(args) -> None:
    import torch

    from paper_2502_10831_b200 import _lib
    from paper_2502_10831_b200.configs import CONFIGS

    ctx = Ctx(args)
    _lib.lib()  # fail loudly if the CUDA library is missing
    w = CONFIGS[args.config]
    head, state = measure(ctx, w, args.steps, args.warmup, args.f32_policy, args.elements, keep=True,
                          burst=not args.no_burst)

    sus = None
    if args.sustained_seconds > 0:
        sus = sustained(ctx, w, state, args.sustained_seconds, head["ms_per_step"], args.f32_policy)

    e2e, e2e_var = None, None
    if not args.no_e2e:
        # the whole shard at N=1; 2^26 per rank at N>1 (N ranks pin N x 2-8 GiB of host memory)
        n_e2e = min(state["n"], args.e2e_elements or (state["n"] if ctx.world == 1 else 1 << 26))
        e2e = e2e_pinned(ctx, w, state, args.e2e_steps, n_e2e)
        e2e_var = e2e_pageable(ctx, w, state, args.e2e_steps, n_e2e) or None

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        from oracle import oracle as O

        threads = O.ncpu()
        if w.dist == 0:
            get = host_inputs(w)
        else:
            xh_all = state["x"].cpu().numpy()
            get = lambda m: xh_all[:m]  # noqa: E731 -- device-generated stress inputs
        rate, kind, ns, sec, _ = cpu_rate(get, w.mask, threads, 10.0)
        cpu = {"value": round(rate, 6), "unit": "Gelem/s", "cores": threads, "kind": kind,
               "sample": f"first {ns} elements of this workload ({sec:.1f} s, one run); fused "
                         f"sin+cos+tan via the scalar reference calls over {threads} threads; "
                         f"{host_cpu_model()}",
               "api_batch_single_thread_gelem_s": api_single_thread_rate(w)}
    del state
    torch.cuda.empty_cache()

    # ---- every other BASELINE config in the same run
    extra = {}
    sel = args.configs
    names = ([] if sel == "none" else [c for c in EXTRA_CONFIGS if c != w.name] if sel == "auto" and w.name == "cfg2"
             else [] if sel == "auto" else [c for c in sel.split(",") if c and c != w.name])
    for c in names:
        k = args.config_steps or CONFIG_STEPS.get(c, 100)
        e, _ = measure(ctx, CONFIGS[c], k, min(args.warmup, 10), args.f32_policy, burst=not args.no_burst)
        extra[c] = e

    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "Gelem/s", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None,
            "dtype": head["dtype"], "data": "synthetic", "config": head["config"],
            "per_gpu_gelem_s": head["per_gpu_gelem_s"], "roofline": head["roofline"],
            "fp64_roof": head["fp64_roof"], "cpu_baseline": cpu, "e2e": e2e, "e2e_variants": e2e_var,
            "gpu_launches": head["gpu_launches"], "clocks": head["clocks"], "burst": head["burst"],
            "aux_kernels": head["aux_kernels"],
            "sustained": sus,
            "accuracy": head["accuracy"],
            "configs": extra or None,
        }
        print(json.dumps(line), flush=True)
    if ctx.dist.is_initialized():
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--configs", default="auto",
                    help="extra configs timed in the same run: auto (all others when --config cfg2), "
                         "none, or a comma list")
    ap.add_argument("--config-steps", type=int, default=0,
                    help="timed steps of every extra config (default: CONFIG_STEPS)")
    ap.add_argument("--elements", type=int, default=0,
                    help="override elements per GPU (weak configs) / of the global array (cfg5)")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="process-group backend; gloo only for tests that run several ranks on one GPU")
    ap.add_argument("--f32-policy", choices=["ulp2", "bitwise"], default="ulp2")
    ap.add_argument("--sustained-seconds", type=float, default=20.0,
                    help="also run the headline step back to back for this long (0: skip)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-elements", type=int, default=0,
                    help="elements per rank per e2e step (default: the whole shard)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-burst", action="store_true", help="skip the short-window (pre-power-cap) timing")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

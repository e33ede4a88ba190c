"""Benchmark of the B200 batched piecewise sin/cos/tan path (arXiv 2502.10831).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

Workload (N=1): BASELINE.json configs[1] -- f64 x, 2^28 elements uniform in
[-1000pi, 1000pi], fused proposed sin+cos+tan (three output arrays), default
SqrtMode (fisr, 1 Newton step).  Under torchrun each rank owns a contiguous
2^28-element shard of one global array (global index = generator counter):
per-GPU work is fixed, so "scaling": "weak".  No element data moves between
GPUs; after the timed region each rank runs the K3 parity/error reduction and
NCCL all-reduces the 64-byte statistics (max / sum), the only collective.

One step = one K1 launch over the shard (inputs already resident in HBM).
Inputs + outputs are 8 GiB per GPU, far above the 126 MB L2, so no flush is
needed between steps.  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.

`e2e` is the same metric through the public host-pointer C-ABI call
(ft_proposed_batch_host) with pinned host buffers: every step copies x in and
sin/cos/tan out (2^26 elements per rank per step by default, so N ranks pin
N x 2 GiB of host memory, not N x 8 GiB; the rate is PCIe-bound either way).  `cpu_baseline` (rank 0, N=1) and `--impl reference` time the
reference's own CPU implementation (oracle/_ref: the unmodified reference
headers, all host threads) on a bounded sample of the same workload.
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


# ------------------------------------------------------------------ reference arm
def run_reference(args) -> None:
    rank = env_int("RANK", 0)
    if rank != 0:
        return  # the reference arm is single-process CPU work; other ranks idle
    import numpy as np

    from oracle import oracle as O
    from paper_2502_10831_b200.configs import CONFIGS

    w = CONFIGS[args.config]
    threads = O.ncpu()
    total_steps = args.steps + args.warmup
    per_step = max(0.2, min(2.0, 120.0 / max(total_steps, 1)))
    # sample inputs: the first elements of the same seeded stream
    rate, kind, n, _, x = cpu_rate(host_inputs(w), w.mask, threads, per_step)
    impl = "ref" if kind == "reference" else "port"
    for _ in range(args.warmup):
        O.proposed(x, w.mask, threads=threads, impl=impl)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.proposed(x, w.mask, threads=threads, impl=impl)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    value = n / (ms / 1e3) / 1e9
    sample = (f"first {n} elements of {w.name} ({w.note}); fused sin+cos+tan via the scalar "
              f"reference calls, contiguous partition over {threads} threads; {host_cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gelem/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if w.itemsize == 8 else "f32", "data": "synthetic",
        "config": {"workload": w.name, "description": w.note, "elements_per_step": n},
        "cpu_baseline": {"value": round(value, 6), "unit": "Gelem/s", "cores": threads,
                         "kind": kind, "sample": sample,
                         "api_batch_single_thread_gelem_s": api_single_thread_rate(w)},
        "e2e": {"value": round(value, 6), "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2502_10831_b200 as ft
    from paper_2502_10831_b200 import _lib
    from paper_2502_10831_b200.configs import CONFIGS, shard
    from paper_2502_10831_b200.dist import reduce_stats

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # torchrun
    if world > 1 or launched:
        dist.init_process_group("nccl", device_id=dev)
    _lib.lib()  # fail loudly if the CUDA library is missing

    w = CONFIGS[args.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    n = args.elements or w.n
    if args.config == "cfg5":
        lo, hi = shard(w.n, rank, world)  # strong: one fixed 2^33 array
        n = hi - lo
        scaling = "strong"
    else:
        lo, hi = rank * n, (rank + 1) * n  # weak: a fixed shard per GPU
        scaling = "weak"
    stream = torch.cuda.current_stream()
    x = ft.gen_inputs(n, tdt, w.dist, w.lo, w.hi, w.seed, lo)
    names = [nm for j, nm in enumerate(("sin", "cos", "tan")) if w.mask & (1 << j)]
    out = {nm: torch.empty_like(x) for nm in names}
    mode = ft.SqrtMode()

    def step():
        if w.kind == 0:
            ft.proposed_eval(x, w.mask, mode, out=out)
        else:
            ft.taylor_eval(x, w.n_terms, w.mask, out=out)

    def barrier():
        if dist.is_initialized():
            dist.barrier()

    clocks = ClockSampler(local)  # samples from warm-up start to timed-region end (GPU loaded)
    clocks.start()
    clocks.mark()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = ft.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = ft.launch_count() - l0
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    elems_total = n * world if scaling == "weak" else w.n
    value = elems_total / (ms / 1e3) / 1e9

    # ---- roofline of the dominant (only) kernel in the step
    peak, peak_src = peaks()
    bytes_per_launch = w.bytes_per_elem * n
    achieved = bytes_per_launch / (ms_local / 1e3) / 1e9

    # ---- accuracy: K3 over the whole shard, NCCL-reduced (max / sum)
    st = ft.parity_reduce(x, out, w.mask, kind=w.kind, mode=mode, n_terms=w.n_terms, ulp_tol=2)
    st = reduce_stats(st, device=dev)  # the path's only collective: 64 B of stats
    accuracy = {
        "checked": int(st["n_checked"]), "max_ulp_vs_oracle": st["max_ulp"],
        "over_2ulp": st["n_over_tol"],
        "max_abs_err_vs_libm": st["max_abs_vs_libm"], "max_rel_err_vs_libm": st["max_rel_vs_libm"],
        "avg_abs_err_vs_libm": [s_ / max(1, c) for s_, c in zip(st["sum_abs_vs_libm"], st["n_finite_libm"])],
        "max_abs_err_vs_oracle": st["max_abs_vs_oracle"], "inf_count": st["n_inf"],
        "nan_count": st["n_nan"], "checksum": st["checksum"], "outputs": names,
        "oracle": "device restatement of the reference (ft_mirror_*), bitwise-pinned to the CPU oracle",
    }

    # ---- e2e through the public host-pointer C-ABI call (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        n_e2e = min(n, args.e2e_elements)
        xh = torch.empty(n_e2e, dtype=tdt, pin_memory=True)
        xh.copy_(x[:n_e2e])
        outs_h = {nm: torch.empty(n_e2e, dtype=tdt, pin_memory=True) for nm in names}
        ptr = [outs_h[nm].data_ptr() if nm in outs_h else None for nm in ("sin", "cos", "tan")]
        L = _lib.lib()
        dtc = _lib.FT_F32 if w.itemsize == 4 else _lib.FT_F64

        def e2e_step():
            if w.kind == 0:
                _lib.check(L.ft_proposed_batch_host(dtc, xh.data_ptr(), n_e2e, w.mask, mode.c(), *ptr))
            else:
                _lib.check(L.ft_taylor_batch_host(dtc, xh.data_ptr(), n_e2e, w.mask, w.n_terms, *ptr))

        e2e_step()  # warm (allocates the pipeline buffers)
        barrier()
        times = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()  # blocking: returns with results in host memory
            times.append(time.perf_counter() - t0)
        te = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_tot = n_e2e * world if scaling == "weak" else n_e2e * world
        e2e = {"value": round(e2e_tot / float(te.item()) / 1e9, 6), "unit": "Gelem/s",
               "h2d_bytes_per_step": n_e2e * w.itemsize,
               "d2h_bytes_per_step": n_e2e * w.itemsize * len(names),
               "elements_per_step_per_gpu": n_e2e, "steps": args.e2e_steps,
               "timing": "host wall clock around the blocking C-ABI call (pinned buffers)"}
        del xh, outs_h

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O

        threads = O.ncpu()
        if w.dist == 0:
            get = host_inputs(w)
        else:
            xh_all = x.cpu().numpy()
            get = lambda m: xh_all[:m]  # noqa: E731 -- device-generated stress inputs
        rate, kind, ns, sec, _ = cpu_rate(get, w.mask, threads, 10.0)
        cpu = {"value": round(rate, 6), "unit": "Gelem/s", "cores": threads, "kind": kind,
               "sample": f"first {ns} elements of this workload ({sec:.1f} s, one run); fused "
                         f"sin+cos+tan via the scalar reference calls over {threads} threads; "
                         f"{host_cpu_model()}",
               "api_batch_single_thread_gelem_s": api_single_thread_rate(w)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "Gelem/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f64" if w.itemsize == 8 else "f32", "data": "synthetic",
            "config": {"workload": w.name, "description": w.note, "elements_per_gpu": n,
                       "outputs": names, "sqrt_mode": "fisr(1) (SqrtMode{} default)",
                       "parallelism": f"dp{world} contiguous shards, no data exchange",
                       "l2": "inputs larger than L2 (x + outputs = "
                             f"{w.bytes_per_elem * n / 2**30:.1f} GiB per GPU vs 126 MB L2); no flush"},
            "per_gpu_gelem_s": round(n / (ms / 1e3) / 1e9, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": ncu_traffic(w.name), "peak_source": peak_src,
                         "algorithmic_bytes_per_elem": w.bytes_per_elem,
                         "kernel": "k_proposed (K1)" if w.kind == 0 else "k_taylor (K2)"},
            "fp64_roof": fp64_roof(w.name, n / (ms / 1e3) / 1e9),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "accuracy": accuracy,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--elements", type=int, default=0, help="override elements per GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-elements", type=int, default=1 << 26,
                    help="elements per rank per e2e step (pinned host buffers of this size)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

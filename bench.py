#!/usr/bin/env python
"""Benchmark of the pk hot path: AG-GEMM + GEMM-RS TFLOP/s (BASELINE.json metric).

One step = one tensor-parallel AG-GEMM followed by one GEMM-RS at
M = N = K = S (default S = 16384, bf16 in / fp32 accumulate / bf16 out):
  AG-GEMM : C_r[S, S/n]  = AllGather(A_r[S/n, S]) @ B_r[S/n, S]^T
  GEMM-RS : out_r[S/n, S] = sum_d (A_d[S, S/n] @ B_d[S, S/n]^T)[rows of r]
Whole-job FLOPs per step = 2 * 2 * S^3 (strong scaling: total work fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--size S] [--impl pk|reference]

N > 1 runs under torchrun (one rank per GPU); the device time is the max over
ranks. Inputs are synthetic (torch.randn * 0.1, seeded per rank) and larger
than L2 (each operand >= 128 MiB at S = 16384), so no L2 flush is needed.
`--impl reference` times the CPU oracle port (oracle/, numpy) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AG-GEMM & GEMM-RS TFLOP/s @1/2/4/8 B200; speedup vs NCCL+cuBLAS non-overlap"
UNIT = "TFLOP/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--size", type=int, default=16384)
    p.add_argument("--impl", default="pk", choices=["pk", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 1590.0, 1400.0, "fallback"


def traffic_for(size: int):
    path = os.path.join(ROOT, "profiles", "gemm_dram_traffic.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get(str(size))
    return None


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_oracle_rate(size: int, seconds: float, slab_div: int = 1):
    """Time the oracle port's AG-GEMM + GEMM-RS (n = 1) in float32 on host cores.

    Returns (TFLOP/s, sample description, threads)."""
    import numpy as np

    import oracle
    rng = np.random.default_rng(0)
    rows = max(1, size // slab_div)
    a = (rng.standard_normal((rows, size)) * 0.1).astype(np.float32)
    b = (rng.standard_normal((size, size)) * 0.1).astype(np.float32)
    flops_per = 2 * 2.0 * rows * size * size
    # every host thread (torchrun exports OMP_NUM_THREADS=1 to each rank, which
    # would otherwise pin the BLAS under the oracle to one core)
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(limits=cpu_threads())
    except Exception:
        limiter = None
    oracle.ag_gemm([a], [b], dtype=np.float32)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.ag_gemm([a], [b], dtype=np.float32)
        oracle.gemm_rs([a], [b], dtype=np.float32)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= seconds:
            break
    if limiter is not None:
        limiter.restore_original_limits()
    tf = flops_per * reps / dt / 1e12
    sample = (f"oracle.ag_gemm + oracle.gemm_rs (numpy float32) at n=1, rows {rows} of M={size}, "
              f"N=K={size}; {reps} steps in {dt:.1f}s")
    return tf, sample, cpu_threads()


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    S = args.size
    n = args.gpus
    # bounded sample: a 1/16 row slab of each GEMM per step
    slab = 16 if S >= 8192 else 1
    import numpy as np

    import oracle
    rng = np.random.default_rng(0)
    rows = S // slab
    a = (rng.standard_normal((rows, S)) * 0.1).astype(np.float32)
    b = (rng.standard_normal((S, S)) * 0.1).astype(np.float32)
    flops = 2 * 2.0 * rows * S * S
    try:                                   # every host thread, even under torchrun's OMP_NUM_THREADS=1
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=cpu_threads())
    except Exception:
        pass
    for _ in range(args.warmup):
        oracle.ag_gemm([a], [b], dtype=np.float32)
        oracle.gemm_rs([a], [b], dtype=np.float32)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.ag_gemm([a], [b], dtype=np.float32)
        oracle.gemm_rs([a], [b], dtype=np.float32)
    dt = time.perf_counter() - t0
    value = flops * args.steps / dt / 1e12
    sample = f"per step: AG-GEMM + GEMM-RS row slab {rows}/{S} rows (numpy float32, oracle port)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"ag_gemm+gemm_rs M=N=K={S} (row-slab sample)", "size": S,
                                        "parallelism": f"tp{n}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_threads(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def l2_note(S: int, n: int) -> str:
    """How the timed loop keeps L2 from carrying data between iterations."""
    op = S * S * 2 / n                                   # one per-rank operand, bytes
    if op > 126e6:
        return f"no flush: every per-rank operand ({op / 1e6:.0f} MB) > L2 (126 MB)"
    # A shard, B, C of the AG-GEMM + the gathered A rows (S x S), and A, B, out of the GEMM-RS
    step = 6 * op + (S * S * 2 if n > 1 else 0)
    if step > 2 * 126e6:
        return (f"no flush: per-rank operands {op / 1e6:.0f} MB, but each step streams {step / 1e6:.0f} MB "
                f"through L2 (126 MB), so no operand is L2-resident when the next iteration reads it")
    return f"warm L2: the step's {step / 1e6:.0f} MB fit in L2 (126 MB); no flush"


def _agree_uid(dist, rank: int, world: int) -> str:
    import uuid
    uid = [uuid.uuid4().hex[:16] if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    return uid[0]



class Watchdog:
    """If the optional legs after the headline measurement hang (a peer that
    never signals, a wedged collective), print what was measured so far and
    exit instead of losing the run."""

    def __init__(self, seconds: float, fire):
        self.t = threading.Timer(seconds, fire)
        self.t.daemon = True

    def start(self):
        self.t.start()

    def cancel(self):
        self.t.cancel()


def _leg(line: dict, key: str, fn):
    """Run one optional leg; its failure is recorded, never fatal to the line."""
    try:
        line[key] = fn()
    except Exception as e:                                  # noqa: BLE001
        line[key] = {"error": f"{type(e).__name__}: {e}"[:400]}


# ----------------------------------------------------------------------------- pk arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2511_13940_b200 as pk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks: all ranks on one GPU (gloo plumbing, no NCCL baseline) to exercise the N>1 path
    if "PK_BENCH_DEVICE" in os.environ:
        local = int(os.environ["PK_BENCH_DEVICE"])
    backend = os.environ.get("PK_BENCH_BACKEND", "nccl")
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
            args.no_baseline = True
        comm = pk.Comm.init(rank, world, local, _agree_uid(dist, rank, world))
    else:
        comm = pk.local_group(1, local)[0]
    n = world
    S = args.size
    if S % (256 * n):
        raise SystemExit(f"--size must be a multiple of {256 * n}")
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)

    def randn(*shape):
        return (torch.randn(*shape, device=dev, generator=g) * 0.1).to(torch.bfloat16)

    # AG-GEMM operands; the shard lives in a symmetric PGL so peers read it in place
    a_ag = comm.empty((S // n, S))
    a_ag.copy_(randn(S // n, S))
    b_ag = randn(S // n, S)
    c_ag = torch.empty(S, S // n, device=dev, dtype=torch.bfloat16)
    # GEMM-RS operands; the output is symmetric so peers reduce-add into it
    a_rs = randn(S, S // n)
    b_rs = randn(S, S // n)
    o_rs = comm.empty((S // n, S))
    flops_step = 2 * 2.0 * S ** 3                  # whole job (all ranks)
    flops_launch = 2.0 * S ** 3 / n                # per rank per GEMM launch
    stream = torch.cuda.current_stream()

    def step(evs=None):
        if evs is not None:
            evs[0].record(stream)
        pk.all_gather_gemm(comm, a_ag, b_ag, out=c_ag)
        if evs is not None:
            evs[1].record(stream)
        pk.gemm_reduce_scatter(comm, a_rs, b_rs, out=o_rs)
        if evs is not None:
            evs[2].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def max_vec(xs: list) -> list:
        if world == 1:
            return list(xs)
        t = torch.tensor(xs, device=dev if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    for _ in range(args.warmup):
        step()
    barrier()
    comm.check()

    # ---------------------------------------------------------------- timed region
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t_end.record(stream)
    barrier()
    clk = clocks.stop()
    comm.check()
    ms_total = max_over_ranks(t_start.elapsed_time(t_end))
    ms_step = ms_total / args.steps
    value = flops_step * args.steps / (ms_total / 1e3) / 1e12
    ag_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    rs_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    launch_ms = max_over_ranks((ag_ms + rs_ms) / 2)

    # ---------------------------------------------------------------- NCCL + cuBLAS, non-overlapped
    base = None
    if not args.no_baseline:
        a_full = torch.empty(S, S, device=dev, dtype=torch.bfloat16) if n > 1 else None
        part = torch.empty(S, S, device=dev, dtype=torch.bfloat16) if n > 1 else None

        def base_step():
            if n > 1:
                dist.all_gather_into_tensor(a_full, a_ag)
                torch.matmul(a_full, b_ag.t(), out=c_ag)
                torch.matmul(a_rs, b_rs.t(), out=part)
                dist.reduce_scatter_tensor(o_rs, part)
            else:
                torch.matmul(a_ag, b_ag.t(), out=c_ag)
                torch.matmul(a_rs, b_rs.t(), out=o_rs)
        for _ in range(args.warmup):
            base_step()
        barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.steps):
            base_step()
        b1.record(stream)
        barrier()
        bms = max_over_ranks(b0.elapsed_time(b1)) / args.steps
        base = {"impl": "torch.matmul (cuBLAS)" + (" + NCCL all_gather / reduce_scatter" if n > 1 else ""),
                "value": flops_step / (bms / 1e3) / 1e12, "ms_per_step": bms, "speedup": bms / ms_step}

    # ---------------------------------------------------------------- end to end (host buffers)
    # Through the public API with pinned host buffers, the copies pipelined
    # against the kernels with double-buffered device tensors: the H2D of step
    # i+1 (copy stream) and the D2H of step i-1 (second copy stream, the other
    # PCIe direction) overlap the fused ops of step i. The weights are layer
    # parameters and stay resident, as in the reference's tensor-parallel layer.
    #   chained (the headline): one tensor-parallel MLP forward per step,
    #     y = gemm_reduce_scatter(all_gather_gemm(x, W1), W2) — the AG-GEMM
    #     output [S, S/n] is the GEMM-RS input (column- then
    #     row-parallel), so only x comes in and y goes out;
    #   separate_ops: the two ops on independent activations, both inputs
    #     copied in and both outputs read back every step.
    e2e = None
    if not args.no_e2e:
        # steady-state throughput: the first step's H2D and the last step's D2H
        # cannot overlap compute, so the e2e loop runs 3x the timed steps
        # (20 -> 60: +2 % e2e, profiles/r2/e2e/bench_k20.json vs bench_k60.json)
        k_e2e = int(os.environ.get("PK_E2E_STEPS", max(4, 3 * args.steps)))
        s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
        nbytes = lambda ts: sum(t.numel() * t.element_size() for t in ts)

        def e2e_measure(chained: bool):
            if chained:
                ins0, outs0 = [a_ag], [o_rs]
                sets = [(ins0, outs0), ([comm.empty(tuple(a_ag.shape))], [comm.empty(tuple(o_rs.shape))])]
            else:
                ins0, outs0 = [a_ag, a_rs], [c_ag, o_rs]
                sets = [(ins0, outs0),
                        ([comm.empty(tuple(a_ag.shape)), torch.empty_like(a_rs)],
                         [torch.empty_like(c_ag), comm.empty(tuple(o_rs.shape))])]
            h_in = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in ins0]
            h_out = [[torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs0] for _ in range(2)]
            for h, t in zip(h_in, ins0):
                h.copy_(t)

            def compute(ins, outs):
                if chained:
                    pk.all_gather_gemm(comm, ins[0], b_ag, out=c_ag)       # c_ag: the intermediate activation
                    pk.gemm_reduce_scatter(comm, c_ag, b_rs, out=outs[0])
                else:
                    pk.all_gather_gemm(comm, ins[0], b_ag, out=outs[0])
                    pk.gemm_reduce_scatter(comm, ins[1], b_rs, out=outs[1])

            def run(k):
                done_compute = [None, None]
                done_d2h = [None, None]
                for i in range(k):
                    ins, outs = sets[i % 2]
                    with torch.cuda.stream(s_h2d):
                        if done_compute[i % 2] is not None:
                            s_h2d.wait_event(done_compute[i % 2])          # step i-2 finished reading this set
                        for t, h in zip(ins, h_in):
                            t.copy_(h, non_blocking=True)
                        ev_in = torch.cuda.Event()
                        ev_in.record(s_h2d)
                    stream.wait_event(ev_in)
                    if done_d2h[i % 2] is not None:
                        stream.wait_event(done_d2h[i % 2])                 # outputs of step i-2 read back
                    compute(ins, outs)
                    ev_c = torch.cuda.Event()
                    ev_c.record(stream)
                    done_compute[i % 2] = ev_c
                    with torch.cuda.stream(s_d2h):
                        s_d2h.wait_event(ev_c)
                        for h, t in zip(h_out[i % 2], outs):
                            h.copy_(t, non_blocking=True)
                        ev_o = torch.cuda.Event()
                        ev_o.record(s_d2h)
                        done_d2h[i % 2] = ev_o
                stream.wait_stream(s_h2d)
                stream.wait_stream(s_d2h)

            run(2)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run(k_e2e)
            e1.record(stream)
            barrier()
            comm.check()
            ems = max_over_ranks(e0.elapsed_time(e1)) / k_e2e
            return {"value": flops_step / (ems / 1e3) / 1e12, "unit": UNIT, "ms_per_step": ems, "steps": k_e2e,
                    "h2d_bytes_per_step": nbytes(ins0), "d2h_bytes_per_step": nbytes(outs0)}

        sep = e2e_measure(False)
        e2e = e2e_measure(True)
        e2e.update({
            "api": "tensor-parallel MLP forward through the public API: y = paper_2511_13940_b200.gemm_reduce_scatter("
                   "all_gather_gemm(x, W1), W2); x copied in from pinned host memory and y read back every step, "
                   "H2D/D2H pipelined against compute (double-buffered device tensors)",
            "resident": "weights W1 (b_ag), W2 (b_rs) and the intermediate activation [S, S/n]",
            "separate_ops": dict(sep, api="all_gather_gemm and gemm_reduce_scatter on independent activations: "
                                          "both inputs copied in, both outputs read back every step"),
        })

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peak_burst, peak_sus, src = peaks()
    achieved = flops_launch / (launch_ms / 1e3) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": UNIT,
                "frac": achieved / peak_burst, "frac_of_sustained_peak": achieved / peak_sus,
                "traffic": traffic_for(S),
                "traffic_source": "ncu --set full, one launch at this size (profiles/gemm_dram_traffic.json)"
                                  if traffic_for(S) else None,
                "kernel": "pk::lcsc_gemm_kernel<2,256,*>",
                "per_launch": f"2*S^3/n = {flops_launch:.4g} FLOP per launch (one AG-GEMM or GEMM-RS)",
                "peak_source": f"{src} bf16_tflops (burst); sustained {peak_sus}",
                "ag_ms": ag_ms, "rs_ms": rs_ms}
    if n > 1:
        # overlapped roofline of one AG-GEMM / GEMM-RS launch (costmodel.py,
        # SURVEY.md §8d): max(compute at peak, link bytes at link bandwidth),
        # against the measured peaks and against the north_star's nominal ones
        from paper_2511_13940_b200 import costmodel as cm
        meas = cm.Profile(name="measured", tensor_R=peak_burst * 1e12, link_B=770e9)
        r_meas, r_nom = cm.ag_gemm(S, n, meas), cm.ag_gemm(S, n, cm.B200_NOMINAL)
        roofline["overlapped"] = {"t_roof_ms": r_meas["t_roof_s"] * 1e3, "limit": r_meas["bound"],
                                  "frac": r_meas["t_roof_s"] * 1e3 / launch_ms,
                                  "t_roof_ms_nominal": r_nom["t_roof_s"] * 1e3,
                                  "frac_nominal": r_nom["t_roof_s"] * 1e3 / launch_ms,
                                  "link_bytes_per_launch": r_meas["link_bytes"], "link_gbs": 770,
                                  "nominal": "2.25 PF/s, 900 GB/s (north_star)"}

    cpu = None
    if rank == 0 and world == 1:
        tf, sample, cores = cpu_oracle_rate(min(S, 4096), args.cpu_seconds)
        cpu = {"value": tf, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    elif rank == 0:
        cpu = {"value": None, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
               "sample": "measured on rank 0 at N=1 only"}

    comm.check()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch.randn*0.1, seeded per rank)",
        "config": {"workload": f"ag_gemm+gemm_rs M=N=K={S} (one AG-GEMM then one GEMM-RS per step)",
                   "size": S, "parallelism": f"tp{n}", "global_batch": S,
                   "l2": l2_note(S, n)},
        "e2e": e2e, "gpu_launches": 2 * args.steps, "roofline": roofline, "cpu_baseline": cpu,
        "nccl_cublas": base, "clocks": clk, "nvls": bool(comm.has_multicast),
    }
    if n > 1:
        # per-op NVLink rate: (n-1)/n of the S x S bf16 operand crosses the
        # links per launch (A rows gathered in, or partial rows reduced out)
        link_bytes = (n - 1) / n * S * S * 2
        ag_max, rs_max = max_over_ranks(ag_ms), max_over_ranks(rs_ms)
        line["link"] = {"bytes_per_launch": link_bytes,
                        "ag_gemm_gbs": link_bytes / (ag_max / 1e3) / 1e9,
                        "gemm_rs_gbs": link_bytes / (rs_max / 1e3) / 1e9,
                        "ag_gemm_frac_of_900": link_bytes / (ag_max / 1e3) / 900e9,
                        "gemm_rs_frac_of_900": link_bytes / (rs_max / 1e3) / 900e9,
                        "note": "algorithmic link bytes / device time of the fused launch (max over ranks)"}

    # ---------------------------------------------------------------- optional legs (never lose the line)
    def emit_and_exit():
        if rank == 0:
            line["watchdog"] = "optional legs did not finish within the limit; line printed as measured so far"
            print(json.dumps(line), flush=True)
        os._exit(0)
    dog = Watchdog(float(os.environ.get("PK_BENCH_LEG_LIMIT_S", "420")), emit_and_exit)
    dog.start()
    _leg(line, "parity", lambda: parity_check(pk, comm, dist, dev, rank, n, S, a_ag, b_ag, c_ag, a_rs, b_rs, o_rs,
                                              max_over_ranks))
    if n > 1:
        _leg(line, "all_reduce", lambda: all_reduce_leg(pk, comm, dist, dev, n, barrier, max_over_ranks,
                                                        backend == "nccl"))
    else:
        line["all_reduce"] = {"skipped": "world 1: an all-reduce is the identity"}
    if n > 1:
        _leg(line, "decomposition", lambda: decomposition_leg(pk, comm, dev, n, S, a_ag, b_ag, c_ag, a_rs, b_rs, o_rs,
                                                              ag_max, rs_max, barrier, max_over_ranks))
    if n > 1:
        _leg(line, "schedule", lambda: schedule_leg(pk, comm, n, S, a_ag, b_ag, c_ag, a_rs, b_rs, o_rs, barrier,
                                                    max_over_ranks))
    _leg(line, "ring_attention", lambda: ring_leg(pk, comm, dist, dev, n, barrier, max_over_ranks,
                                                  backend == "nccl", args.size))
    _leg(line, "moe", lambda: moe_leg(pk, comm, dist, dev, n, barrier, max_over_ranks, backend == "nccl"))
    _leg(line, "nvlink", lambda: nvlink_leg(comm, n, barrier, max_vec))
    dog.cancel()
    comm.check()
    ok = not any(isinstance(line.get(key), dict) and line[key].get("ok") is False
                 for key in ("parity", "ring_attention", "moe"))
    if rank == 0:
        print(json.dumps(line), flush=True)
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0 if ok else 1


# ----------------------------------------------------------------------------- optional legs
def parity_check(pk, comm, dist, dev, rank, n, S, a_ag, b_ag, c_ag, a_rs, b_rs, o_rs, max_over_ranks) -> dict:
    """Exact integer-data parity of the two timed ops at the timed size, on
    every rank, against an independent path: NCCL all-gather / reduce-scatter
    plus an fp32 torch GEMM (integer sums below 2^24 are exact in fp32, so the
    bf16-rounded results must match bit for bit). GEMM-RS inputs are nonzero
    in only 256/n columns of K, so every partial and every running sum of the
    cross-rank bf16 reduce-add stays within bf16's exact integers (|x| <= 256)."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(4321 + rank)

    def ints(shape, lo, hi):
        return torch.randint(lo, hi + 1, shape, device=dev, generator=g).to(torch.bfloat16)

    out = {"inputs": "integers: AG-GEMM A, B in [-2, 2]; GEMM-RS A, B in [-1, 1], A nonzero in 256/n K columns",
           "reference": "NCCL all_gather / reduce_scatter + cuBLAS bf16 GEMM (fp32 accumulation, no reduced-"
                        "precision split-K reduction): every sum is an exact integer, rounded to bf16 once"}
    prev = torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    a_ag.copy_(ints(tuple(a_ag.shape), -2, 2))
    b_ag.copy_(ints(tuple(b_ag.shape), -2, 2))
    pk.all_gather_gemm(comm, a_ag, b_ag, out=c_ag)
    nccl = dist.is_initialized() and dist.get_backend() == "nccl"
    if n > 1 and nccl:
        full = torch.empty(S, S, device=dev, dtype=torch.bfloat16)
        dist.all_gather_into_tensor(full, a_ag)
    elif n > 1:                                   # gloo test plumbing: gather on the host
        parts = [torch.empty(tuple(a_ag.shape), dtype=torch.bfloat16) for _ in range(n)]
        dist.all_gather(parts, a_ag.cpu())
        full = torch.cat(parts).to(dev)
    else:
        full = a_ag
    ref = full @ b_ag.t()
    del full
    bad_ag = int((c_ag != ref).sum().item())
    del ref
    k_loc = a_rs.shape[1]
    a_rs.zero_()
    a_rs[:, :max(1, min(k_loc, 256 // n))] = ints((S, max(1, min(k_loc, 256 // n))), -1, 1)
    b_rs.copy_(ints(tuple(b_rs.shape), -1, 1))
    pk.gemm_reduce_scatter(comm, a_rs, b_rs, out=o_rs)
    part = a_rs @ b_rs.t()                          # |partial| <= 256 / n: exact in bf16
    if n > 1 and nccl:
        red = torch.empty(S // n, S, device=dev, dtype=torch.bfloat16)
        dist.reduce_scatter_tensor(red, part)
    elif n > 1:
        host = part.float().cpu()
        dist.all_reduce(host)
        red = host[rank * (S // n):(rank + 1) * (S // n)].to(dev)
    else:
        red = part
    bad_rs = int((o_rs != red.to(torch.bfloat16)).sum().item())
    del part, red
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = prev
    torch.cuda.synchronize()
    comm.check()
    bad = max_over_ranks(float(bad_ag + bad_rs))
    bad_ag_all, bad_rs_all = max_over_ranks(float(bad_ag)), max_over_ranks(float(bad_rs))
    out.update({"ag_gemm_mismatches": int(bad_ag_all), "gemm_rs_mismatches": int(bad_rs_all),
                "elements_checked_per_rank": int(c_ag.numel() + o_rs.numel()), "ok": bad == 0})
    return out


def all_reduce_leg(pk, comm, dist, dev, n, barrier, max_over_ranks, with_nccl: bool) -> dict:
    """NVLS (or P2P) all-reduce at 64 MiB and 1 GiB per rank, bf16, in a
    symmetric (multicast when available) buffer; exactness checked on integer
    data first; NCCL all_reduce of the same size alongside. algbw = bytes / t
    (the NVLS roofline moves ~S per direction per GPU)."""
    import torch
    rank = comm.rank
    res = {"path": "nvls (multimem.ld_reduce + multimem.st)" if comm.has_multicast else "p2p register ops",
           "sizes": []}
    cap = int(os.environ.get("PK_BENCH_AR_MAX_BYTES", str(1 << 30)))      # test hook: smaller sizes
    for nbytes, iters in ((64 << 20, 20), (1 << 30, 5)):
        if nbytes > cap:
            continue
        numel = nbytes // 2
        x = comm.empty((numel,), torch.bfloat16, multicast=comm.has_multicast)
        idx = torch.arange(numel, device=dev, dtype=torch.int32) % 17 - 8
        x.copy_((idx + rank % 4).to(torch.bfloat16))
        pk.all_reduce(comm, x)
        exp = (idx * n + sum(r % 4 for r in range(n))).to(torch.bfloat16)
        bad = max_over_ranks(float((x != exp).sum().item()))
        del idx, exp
        pk.all_reduce(comm, x)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            pk.all_reduce(comm, x)
        e1.record()
        barrier()
        comm.check()
        t = max_over_ranks(e0.elapsed_time(e1) / iters) / 1e3
        algbw = nbytes / t
        ent = {"bytes_per_rank": nbytes, "ms": t * 1e3, "algbw_gbs": algbw / 1e9,
               "busbw_gbs": algbw * 2 * (n - 1) / n / 1e9, "frac_of_900": algbw / 900e9,
               "exact_on_integers": bad == 0, "iters": iters}
        if with_nccl:
            y = torch.zeros(numel, device=dev, dtype=torch.bfloat16)
            dist.all_reduce(y)
            barrier()
            e0.record()
            for _ in range(iters):
                dist.all_reduce(y)
            e1.record()
            barrier()
            tn = max_over_ranks(e0.elapsed_time(e1) / iters) / 1e3
            ent["nccl_ms"] = tn * 1e3
            ent["speedup_vs_nccl"] = tn / t
            del y
        res["sizes"].append(ent)
        x._pk_pgl.free()
        del x
    return res


def decomposition_leg(pk, comm, dev, n, S, a_ag, b_ag, c_ag, a_rs, b_rs, o_rs, ag_ms, rs_ms, barrier,
                      max_over_ranks) -> dict:
    """The paper's time decomposition (lcsc.py:110-138) of the
    two fused ops, measured: the compute-only twin (the same per-rank GEMM
    with no communication), the communication-only twin (pk all-gather of the
    A shards / pk reduce-scatter of a bf16 partial) and the non-overlapped
    residual t_fused - max(t_comp, t_comm); comm_ratio = (t_fused - t_comp) /
    t_fused, the paper's non-overlapped communication ratio."""
    import torch

    def timed(fn, iters=5):
        fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / iters)
    full = comm.empty((S, S))            # symmetric: the reduce-scatter twin reads peers' partials in place
    out = {}
    t_comp = timed(lambda: pk.gemm(full, b_ag, out=c_ag))
    t_comm = timed(lambda: pk.all_gather(comm, a_ag, out=full))
    out["ag_gemm"] = {"t_fused_ms": ag_ms, "t_comp_ms": t_comp, "t_comm_ms": t_comm,
                      "t_non_overlap_ms": max(0.0, ag_ms - max(t_comp, t_comm)),
                      "comm_ratio": max(0.0, (ag_ms - t_comp) / ag_ms)}
    t_comp = timed(lambda: pk.gemm(a_rs, b_rs, out=full))
    part = torch.empty(S // n, S, device=dev, dtype=torch.bfloat16)
    t_comm = timed(lambda: pk.reduce_scatter(comm, full, out=part))
    out["gemm_rs"] = {"t_fused_ms": rs_ms, "t_comp_ms": t_comp, "t_comm_ms": t_comm,
                      "t_non_overlap_ms": max(0.0, rs_ms - max(t_comp, t_comm)),
                      "comm_ratio": max(0.0, (rs_ms - t_comp) / rs_ms)}
    full._pk_pgl.free()
    del full, part
    comm.check()
    return out


def schedule_leg(pk, comm, n, S, a_ag, b_ag, c_ag, a_rs, b_rs, o_rs, barrier, max_over_ranks) -> dict:
    """The reference's autotune_partition (lcsc.py:164-191) on the real ranks:
    intra-SM, hybrid (communicator warps) and inter-SM with several
    communicator-SM counts for AG-GEMM, and
    intra-SM (bf16 / fp32 partials) vs inter-SM for GEMM-RS, at the timed
    size; device time max over ranks; ties toward fewer communicator SMs. The
    `table` entry is a measured schedule table (tune.ScheduleTable format)."""
    import torch

    from paper_2511_13940_b200 import tune

    def timed(fn, iters=3):
        fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / iters)
    out = {"size": S, "world": n}
    table = tune.ScheduleTable()
    ag_c = [{"mode": "intra_sm"}, {"mode": "hybrid"}] + [{"mode": "inter_sm", "num_comm_sms": k} for k in (4, 8, 16, 24)]
    rows = [(sc, timed(lambda: pk.all_gather_gemm(comm, a_ag, b_ag, out=c_ag, schedule=sc))) for sc in ag_c]
    best, t = tune.pick_best(rows)
    table.put("ag_gemm", n, S, S, S, best, ms=round(t, 4), emulated=False, sms_per_rank=comm.num_sms)
    out["ag_gemm"] = {"rows": [[sc, ms] for sc, ms in rows], "best": best}
    rs_c = [{"mode": "intra_sm"}, {"mode": "intra_sm", "partials": "fp32"}, {"mode": "inter_sm", "num_comm_sms": 16}]
    rows = [(sc, timed(lambda: pk.gemm_reduce_scatter(comm, a_rs, b_rs, out=o_rs, schedule=sc))) for sc in rs_c]
    best, t = tune.pick_best(rows)
    table.put("gemm_rs", n, S, S, S, best, ms=round(t, 4), emulated=False, sms_per_rank=comm.num_sms)
    out["gemm_rs"] = {"rows": [[sc, ms] for sc, ms in rows], "best": best}
    out["table"] = table.entries
    comm.check()
    return out


def _gather0(dist, t, n: int, nccl: bool):
    """Rank-major concatenation of every rank's t along dim 0 (NCCL, or gloo on the host)."""
    import torch
    if n == 1:
        return t
    if nccl:
        out = torch.empty((n * t.shape[0],) + tuple(t.shape[1:]), device=t.device, dtype=t.dtype)
        dist.all_gather_into_tensor(out, t.contiguous())
        return out
    parts = [torch.empty(tuple(t.shape), dtype=t.dtype) for _ in range(n)]
    dist.all_gather(parts, t.cpu())
    return torch.cat(parts).to(t.device)


def ring_leg(pk, comm, dist, dev, n, barrier, max_over_ranks, nccl: bool, S_gemm: int) -> dict:
    """BASELINE config 4 on this run's ranks: ring attention B1 H16 D128,
    non-causal, S = 32768 and 131072 split over the ranks (the 2-slot device
    ring; n = 1 is the single-GPU kernel). Parity: 16 sampled query rows per
    rank against float64 softmax over every key (K/V gathered with NCCL),
    |o| <= 2e-2, |lse| <= 1e-3 * max(1, |lse|). Whole-job TFLOP/s; the
    non-overlapped baseline is NCCL all-gather of K and V then torch SDPA."""
    import torch
    out = {"B": 1, "H": 16, "D": 128, "sizes": []}
    if S_gemm < 16384:                                # small test runs: small attention too
        sizes = (8192,)
    else:
        sizes = (32768, 131072)
    for S in sizes:
        sl = S // n
        g = torch.Generator(device=dev)
        g.manual_seed(77 + comm.rank)
        q = torch.randn(1, sl, 16, 128, device=dev, generator=g).bfloat16()
        k = comm.empty((1, sl, 16, 128))
        v = comm.empty((1, sl, 16, 128))
        k.copy_(torch.randn(k.shape, device=dev, generator=g).bfloat16())
        v.copy_(torch.randn(v.shape, device=dev, generator=g).bfloat16())
        o, lse = pk.ring_attention(comm, q, k, v)
        torch.cuda.synchronize()
        comm.check()
        K_ = _gather0(dist, k[0], n, nccl).double()
        V_ = _gather0(dist, v[0], n, nccl).double()
        rows = torch.randint(0, sl, (16,), device=dev, generator=g)
        sc = torch.einsum("qhd,khd->hqk", q[0, rows].double(), K_) * 128 ** -0.5
        ref_l = torch.logsumexp(sc, -1)
        ref_o = torch.einsum("hqk,khd->qhd", torch.softmax(sc, -1), V_)
        err_o = max_over_ranks((o[0, rows].double() - ref_o).abs().max().item())
        err_l = max_over_ranks((lse[0][:, rows].double() - ref_l).abs().max().item())
        lim_l = 1e-3 * max(1.0, ref_l.abs().max().item())
        del K_, V_, sc, ref_o

        def timed(fn, iters):
            fn()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            barrier()
            return max_over_ranks(e0.elapsed_time(e1) / iters)
        iters = 3 if S <= 32768 else 2
        t = timed(lambda: pk.ring_attention(comm, q, k, v, out=o, lse=lse), iters)
        flops = n * 4.0 * 16 * sl * S * 128
        ent = {"S": S, "ms": t, "tflops": flops / t / 1e9, "max_err_o": err_o, "max_err_lse": err_l,
               "ok": err_o <= 2e-2 and err_l <= lim_l, "link_bytes_per_rank": (n - 1) * 2 * sl * 16 * 128 * 2}
        if n > 1:
            ent["link_gbs"] = ent["link_bytes_per_rank"] / (t / 1e3) / 1e9
        if nccl and n > 1:
            def base():
                K2 = _gather0(dist, k[0], n, True)
                V2 = _gather0(dist, v[0], n, True)
                torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2), K2[None].transpose(1, 2),
                                                                 V2[None].transpose(1, 2))
            tb = timed(base, iters)
            ent["nccl_sdpa_ms"] = tb
            ent["speedup_vs_nccl_sdpa"] = tb / t
        out["sizes"].append(ent)
        k._pk_pgl.free()
        v._pk_pgl.free()
        del q, k, v, o, lse
    out["ok"] = all(e["ok"] for e in out["sizes"])
    return out


def moe_leg(pk, comm, dist, dev, n, barrier, max_over_ranks, nccl: bool) -> dict:
    """BASELINE config 5 on this run's ranks: 64 experts, top-8, H 7168,
    H_exp 2048, T 4096 tokens per rank, expert e on rank e % n (workloads.py:
    799-802 routing). Dispatch (expert-major) -> planned grouped GEMM1 ->
    combine of the dispatched rows. Parity: every received row is the token
    its id names (tokens gathered with NCCL), counts add up to n * T * k, and
    combine with weights 1/k returns every token exactly."""
    import torch
    T, E, K, H, HE = 4096, 64, 8, 7168, 2048
    g = torch.Generator(device=dev)
    g.manual_seed(99 + comm.rank)
    x = torch.randint(-8, 9, (T, H), device=dev, generator=g).bfloat16()
    topk = torch.rand(T, E, device=dev, generator=g).argsort(1)[:, :K].int().contiguous()
    le = (E + n - 1) // n
    w = (torch.randn(le, HE, H, device=dev, generator=g) * 0.02).bfloat16()
    recv, src, cnt, plan = pk.moe_dispatch(comm, x, topk, E, layout="expert")
    torch.cuda.synchronize()
    comm.check()
    allx = _gather0(dist, x, n, nccl)
    ids = src[:, 0].long()
    real = ids >= 0
    rows_ok = bool(torch.equal(recv[real], allx[ids[real] // K]))
    t_all = torch.tensor([float(int(cnt.item()))], device=dev if nccl else "cpu", dtype=torch.float64)
    if n > 1:
        dist.all_reduce(t_all)
    counts_ok = int(t_all.item()) == n * T * K
    y = pk.grouped_gemm(recv, None, w, plan=plan)
    comb = pk.moe_combine(comm, recv, topk, torch.full((T, K), 1.0 / K, device=dev), E)
    torch.cuda.synchronize()
    comm.check()
    comb_ok = bool(torch.equal(comb, x))
    del allx

    def timed(fn, iters=5):
        fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / iters)
    t_d = timed(lambda: pk.moe_dispatch(comm, x, topk, E, recv=(recv, src), layout="expert"))
    t_g = timed(lambda: pk.grouped_gemm(recv, None, w, out=y, plan=plan))
    t_c = timed(lambda: pk.moe_combine(comm, recv, topk, torch.full((T, K), 1.0 / K, device=dev), E, out=comb))
    rows_moved = T * K                                   # per rank, both directions
    link = rows_moved * (n - 1) / n * H * 2
    out = {"T": T, "E": E, "top_k": K, "H": H, "H_expert": HE, "dispatch_ms": t_d, "grouped_gemm1_ms": t_g,
           "combine_ms": t_c, "rows_ok": rows_ok, "counts_ok": counts_ok, "combine_exact": comb_ok,
           "gemm1_tflops_per_rank": 2.0 * int(cnt.item()) * H * HE / (t_g / 1e3) / 1e12,
           "ok": rows_ok and counts_ok and comb_ok}
    if n > 1:
        out["dispatch_link_gbs"] = link / (t_d / 1e3) / 1e9
        out["combine_link_gbs"] = link / (t_c / 1e3) / 1e9
    return out


def nvlink_leg(comm, n, barrier, max_vec) -> dict:
    """Transfer-mechanism calibration (mechanisms.py / pk_mech_probe): GB/s
    over message size and SM count for the copy engine, TMA, register ops and
    multimem, every rank pushing to rank + 1 at once. One GPU: loopback only."""
    from paper_2511_13940_b200 import mechanisms
    if n == 1:
        res = mechanisms.measure(comm, nbytes=64 << 20, quick=True, reps=2)
        return {"skipped": "one GPU: no NVLink to measure", "loopback_peak_gbs": res["peak_gbs"],
                "loopback_sms_to_saturate": res["sms_to_saturate"]}

    return mechanisms.measure(comm, barrier, max_vec, nbytes=128 << 20, reps=3)


if __name__ == "__main__":
    sys.exit(main())

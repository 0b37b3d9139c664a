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
    # Through the public API with pinned host buffers: every step copies its
    # two activation inputs (the AG-GEMM shard and the GEMM-RS input) host ->
    # device and reads both full outputs back; the two weight matrices are
    # layer parameters and stay resident, as in the reference's tensor-parallel
    # layer. The copies are pipelined against the kernels with double-buffered
    # device tensors: the H2D of step i+1 (copy stream) and the D2H of step i-1
    # (second copy stream, the other PCIe direction) overlap the fused ops of
    # step i.
    e2e = None
    if not args.no_e2e:
        ins0 = [a_ag, a_rs]
        outs0 = [c_ag, o_rs]
        sets = [(ins0, outs0),
                ([comm.empty(tuple(a_ag.shape)), torch.empty_like(a_rs)],
                 [torch.empty_like(c_ag), comm.empty(tuple(o_rs.shape))])]
        h_in = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in ins0]
        h_out = [[torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs0] for _ in range(2)]
        for h, t in zip(h_in, ins0):
            h.copy_(t)
        k_e2e = max(4, args.steps)          # enough steps that the unoverlapped first H2D / last D2H amortise
        s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()

        def e2e_run(k):
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
                pk.all_gather_gemm(comm, ins[0], b_ag, out=outs[0])
                pk.gemm_reduce_scatter(comm, ins[1], b_rs, out=outs[1])
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

        e2e_run(2)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_run(k_e2e)
        e1.record(stream)
        barrier()
        comm.check()
        ems = max_over_ranks(e0.elapsed_time(e1)) / k_e2e
        e2e = {"value": flops_step / (ems / 1e3) / 1e12, "unit": UNIT, "ms_per_step": ems, "steps": k_e2e,
               "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in ins0),
               "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in outs0),
               "api": "paper_2511_13940_b200.all_gather_gemm + gemm_reduce_scatter, pinned host buffers, "
                      "H2D/D2H pipelined against compute (double-buffered device tensors)",
               "resident": "weights b_ag, b_rs (layer parameters); activations copied in, outputs copied out every step"}

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peak_burst, peak_sus, src = peaks()
    achieved = flops_launch / (launch_ms / 1e3) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": UNIT,
                "frac": achieved / peak_burst, "frac_of_sustained_peak": achieved / peak_sus,
                "traffic": traffic_for(S),
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
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch.randn*0.1, seeded per rank)",
            "config": {"workload": f"ag_gemm+gemm_rs M=N=K={S} (one AG-GEMM then one GEMM-RS per step)",
                       "size": S, "parallelism": f"tp{n}", "global_batch": S,
                       "l2": l2_note(S, n)},
            "e2e": e2e, "gpu_launches": 2 * args.steps, "roofline": roofline, "cpu_baseline": cpu,
            "nccl_cublas": base, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Power-cap experiment: does the 16384^3 GEMM lose throughput when it runs on
fewer SMs? (the clock rises under the same ~1 kW cap). cuBLAS's nvjet kernel
for this shape uses 4-CTA clusters (2 pairs, A multicast) that fit 132 SMs.
Prints ms, TF/s, W, MHz and J per GEMM for cuBLAS and pk.gemm at several SM
counts (schedule num_sms)."""
import os, sys, json, time, threading
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import pynvml
import paper_2511_13940_b200 as pk

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
S = int(os.environ.get("S", 16384))
a = torch.randn(S, S, device="cuda").bfloat16() * 0.1
b = torch.randn(S, S, device="cuda").bfloat16() * 0.1
c = torch.empty(S, S, device="cuda", dtype=torch.bfloat16)
configs = [("cublas", lambda: torch.matmul(a, b.t(), out=c))]
for n in [int(x) for x in os.environ.get("SMS", "148,140,132,124,116").split(",")]:
    configs.append((f"pk_{n}", (lambda n=n: pk.gemm(a, b, c, schedule={"num_sms": n}))))


def run(name, fn, seconds=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1e3, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            time.sleep(0.02)
    th = threading.Thread(target=sampler)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(10, int(seconds / 0.006))
    th.start()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    s = samples[len(samples) // 4:]
    pw = sorted(x[0] for x in s)[len(s) // 2]
    clk = sorted(x[1] for x in s)[len(s) // 2]
    r = dict(cfg=name, ms=round(ms, 4), tflops=round(2 * S ** 3 / ms / 1e9, 1), watts=round(pw, 1), mhz=clk,
             joules=round(pw * ms / 1e3, 4))
    print(json.dumps(r), flush=True)
    return r


os.makedirs("gpurun_out", exist_ok=True)
out = os.environ.get("OUT", "gpurun_out/gemm_sms_power.jsonl")
with open(out, "w") as f:
    for rep in range(int(os.environ.get("REPS", 2))):
        for name, fn in configs:
            f.write(json.dumps(run(name, fn)) + "\n")

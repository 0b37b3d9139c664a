"""GEMM energy experiment: ms, SM clock, power and J per 16384^3 GEMM for
cuBLAS and several LCSC kernel configurations (tuning hooks via env)."""
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

configs = [
    ("cublas", {}, lambda: torch.matmul(a, b.t(), out=c)),
    ("pk_am1_m8", {"PK_RASTER": "0,8"}, lambda: pk.gemm(a, b, c)),
    ("pk_am1_m4", {"PK_RASTER": "0,4"}, lambda: pk.gemm(a, b, c)),
    ("pk_am1_s8", {"PK_RASTER": "2,8"}, lambda: pk.gemm(a, b, c)),
    ("pk_am2_m8", {"PK_RASTER": "0,8", "PK_GEMM_AM": "2"}, lambda: pk.gemm(a, b, c)),
    ("pk_am2_m4", {"PK_RASTER": "0,4", "PK_GEMM_AM": "2"}, lambda: pk.gemm(a, b, c)),
    ("pk_am2_s4", {"PK_RASTER": "2,4", "PK_GEMM_AM": "2"}, lambda: pk.gemm(a, b, c)),
    ("pk_am2_s8", {"PK_RASTER": "2,8", "PK_GEMM_AM": "2"}, lambda: pk.gemm(a, b, c)),
]
extra = os.environ.get("EXTRA_CONFIGS")
if extra:
    for name, env in json.loads(extra):
        configs.append((name, env, lambda: pk.gemm(a, b, c)))


def run(name, env, fn, seconds=3.0):
    for k in ("PK_RASTER", "PK_GEMM_AM", "PK_EPI_DIRECT", "PK_L2PROMO"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1e3,
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
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
             joules=round(pw * ms / 1e3, 4), flop_per_clk_sm=round(2 * S ** 3 / (ms / 1e3) / (clk * 1e6) / 148, 1))
    print(json.dumps(r), flush=True)
    return r


os.makedirs("gpurun_out", exist_ok=True)
res = []
for rep in range(int(os.environ.get("REPS", 2))):
    for name, env, fn in configs:
        res.append(run(name, env, fn))
with open("gpurun_out/gemm_power.jsonl", "w") as f:
    for r in res:
        f.write(json.dumps(r) + "\n")

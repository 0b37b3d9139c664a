"""Attention energy probe: ms, SM clock, power, J and SM cycles per call for
the library's attention (PK_LIB selects the build) and torch SDPA, each run
back to back for a few seconds with NVML sampled alongside. Separates a
kernel that needs more cycles from one that runs at a lower clock under the
power cap."""
import os, sys, json, time, threading
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import pynvml
import paper_2511_13940_b200 as pk

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
lib = os.environ.get("PK_LIB", "libpk.so").split("/")[-1] + "".join("+" + k[8:].lower() for k in sorted(os.environ) if k.startswith("PK_ATTN_"))
out = open(sys.argv[1], "a") if len(sys.argv) > 1 else sys.stdout


def run(name, fn, flops, seconds=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    n = max(5, int(seconds * 1e3 / max(e0.elapsed_time(e1), 1e-3)))
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1e3, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            time.sleep(0.02)
    th = threading.Thread(target=sampler)
    th.start()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / n
    s = samples[len(samples) // 4:] or samples
    pw = sorted(x[0] for x in s)[len(s) // 2]
    mhz = sorted(x[1] for x in s)[len(s) // 2]
    rec = dict(lib=lib, op=name, ms=ms, tflops=flops / ms / 1e9, sm_mhz=mhz, power_w=pw, joule=pw * ms / 1e3,
               mcycles=ms * mhz / 1e3)
    out.write(json.dumps(rec) + "\n"); out.flush()


torch.manual_seed(0)
for Sq, Skv in ((16384, 16384), (8192, 65536)):
    q = torch.randn(1, Sq, 16, 128, device="cuda").bfloat16()
    k = torch.randn(1, Skv, 16, 128, device="cuda").bfloat16()
    v = torch.randn_like(k)
    o, lse = torch.empty_like(q), torch.empty(1, 16, Sq, device="cuda")
    flops = 4 * 16 * Sq * Skv * 128
    run(f"pk_attention_q{Sq}_kv{Skv}", lambda: pk.attention(q, k, v, out=o, lse=lse), flops)
    if os.environ.get("SDPA", "1") == "1":
        qt, kt, vt = (x.transpose(1, 2).contiguous() for x in (q, k, v))
        run(f"sdpa_q{Sq}_kv{Skv}", lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt), flops)

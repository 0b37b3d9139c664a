"""Where the device-staged ring spends its time (AT_RING_PROF build):
    PK_BUILD_DEFINES=-DAT_RING_PROF python -m paper_2511_13940_b200.build
    PK_LIB=paper_2511_13940_b200/libpk_DAT_RING_PROF.so python profiles/ring_prof.py
Counters are summed clock64 cycles over threads that own each role; printed
per compute CTA (or per communicator CTA) as fractions of a CTA's lifetime."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from paper_2511_13940_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    buf = (ctypes.c_ulonglong * 12)()
    for n, S in ((2, 32768), (8, 32768), (8, 131072)):
        B, H, D = 1, 16, 128
        sl = S // n
        comms = pk.local_group(n)
        g = torch.Generator(device="cuda").manual_seed(0)
        qs = [torch.randn(B, sl, H, D, device="cuda", generator=g).bfloat16() for _ in comms]
        ks = [c.empty((B, sl, H, D)) for c in comms]
        vs = [c.empty((B, sl, H, D)) for c in comms]
        for t in ks + vs:
            t.copy_(torch.randn(t.shape, device="cuda", generator=g).bfloat16())
        outs = [(torch.empty_like(q), torch.empty(B, H, sl, device="cuda")) for q in qs]
        streams = [torch.cuda.Stream() for _ in comms]

        def ring():
            torch.cuda.synchronize()
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    pk.ring_attention(c, qs[r], ks[r], vs[r], out=outs[r][0], lse=outs[r][1], stream=streams[r])
            torch.cuda.synchronize()
        ring()
        lib.pk_debug_ring_prof(buf, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ring()
        e1.record()
        torch.cuda.synchronize()
        lib.pk_debug_ring_prof(buf, 0)
        v = list(buf)
        ncomm = None
        items = B * H * (sl // 256)
        units = v[4]
        ctas = max(1, v[7] and round(v[7] / max(1, v[7] / (units or 1))))
        life = v[7]                                 # summed over compute CTAs
        out = {"world": n, "S": S, "ms": e0.elapsed_time(e1), "units": units, "items_per_step": items,
               "loader_slot_wait_frac": v[0] / life, "merge_wait_frac(warp-lane0 sum / 8 warps)": v[1] / life / 8,
               "epilogue_frac(per warp)": v[2] / life / 8, "mma_q_wait_frac": v[3] / life,
               "epi_o_full_wait_frac": v[8] / life / 8, "epi_drain_merge_frac": v[9] / life / 8,
               "epi_state_store_frac": v[10] / life / 8,
               "comm_slot_wait_cycles": v[5], "comm_copy_cycles": v[6], "cta_lifetime_cycles_sum": life}
        print(json.dumps(out), flush=True)
        for c in comms:
            c.check()
            c.destroy()


if __name__ == "__main__":
    main()

"""Small ring-attention calls for compute-sanitizer runs: comm warps and comm
CTAs, spans 1 / 2 / whole ring, emulated n = 2 / 4 / 8, checked vs the oracle."""
import os, sys
ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_ring_attention import run  # noqa: E402

for world, sched in ((2, None), (4, {"stages": 4}), (8, None), (8, {"stages": 16}), (4, {"mode": "inter_sm"})):
    run(world, 1, 256, 2, seed=world, schedule=sched)
    print("ok", world, sched, flush=True)

"""Multi-process host logic of the N>1 path, on CPU (no GPU needed).

* pk_debug_rendezvous: every rank of a world-2/4 process group runs the same
  abstract-Unix-socket rendezvous that pk_comm_init uses (rank-id allgather,
  barrier, SCM_RIGHTS exchange of file descriptors — the path VMM handles
  take between torchrun ranks).
* the rendezvous uid is agreed through torch.distributed (gloo), as in
  Comm.init_from_env / bench.py under torchrun.
"""
import os
import socket
import uuid

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = [uuid.uuid4().hex[:16] if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    from paper_2511_13940_b200 import _lib
    lib = _lib.load()
    st = lib.pk_debug_rendezvous(rank, world, uid[0].encode())
    msg = "" if st == 0 else _lib.last_error()
    # max over ranks of the status, like bench.py's max-over-ranks timing
    import torch
    t = torch.tensor([st], dtype=torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    with open(os.path.join(result_dir, f"r{rank}"), "w") as f:
        f.write(f"{st} {int(t.item())} {msg}")
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_rendezvous_multiprocess(world, tmp_path, libpk):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        st, mx, *msg = open(tmp_path / f"r{r}").read().split(" ", 2)
        assert st == "0" and mx == "0", (r, msg)


def test_rendezvous_rejects_bad_world(libpk):
    from paper_2511_13940_b200 import _lib
    assert libpk.pk_debug_rendezvous(0, 1, b"x") == _lib.PK_ERR_INVALID

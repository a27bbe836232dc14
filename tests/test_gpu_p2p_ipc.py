"""The multi-process setup of the peer exchange (sharding.P2PExchange.create): two processes on one GPU exchange
CUDA IPC handles of their arenas over a gloo group and store into each other's arena with the library's kernels.

No kernel here waits on another process's kernel while it runs (the guide's rule for one GPU): each owner's
kd_p2p_combine sees its arrival target (0) already met, and kd_p2p_wait is launched only after a host barrier that
follows both processes' combines, so its done target is met when it starts.  Checked: the rows each owner stores
into the PEER's dh_out / loss_out through the IPC mapping arrive (every row of both arenas is written by exactly one
of the two processes), and both ranks' done counters reach 1."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2603_01875_b200 import kdfused
        from paper_2603_01875_b200.sharding import P2PExchange
        n, d_s = 10, 64  # 5 rows owned per rank
        ex = P2PExchange.create(None, d_s, max_rows=16, max_tokens=32)
        dh, ls = kdfused.p2p_outputs(ex.x, "cuda:0", n, d_s)
        dh.fill_(7.0)
        ls.fill_(7.0)
        torch.cuda.synchronize()
        dist.barrier()
        kdfused.p2p_combine(ex.x, 0, n, 0, None, with_loss=True, target=0)  # zero slots: zero rows everywhere
        torch.cuda.synchronize()
        dist.barrier()
        kdfused.p2p_wait(ex.x, 1)  # both owners' done counters are already 1
        torch.cuda.synchronize()
        q.put((rank, float(dh.abs().max().item()), float(ls.abs().max().item()), len(ex.mapped)))
        dist.barrier()
        ex.close()
    finally:
        dist.destroy_process_group()


def test_p2p_exchange_ipc_two_processes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, dh_max, ls_max, n_mapped in res:
        assert n_mapped == 1
        assert dh_max == 0.0 and ls_max == 0.0, f"rank {rank}: rows the peer owns did not arrive"

"""Failure handling of the ring transport: a peer that
never sends must not block a rank forever.  gloo, world 2, CPU."""

import os
import socket
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2411_01783_b200.ring import TorchRingComm

    comm = TorchRingComm(timeout_s=2.0)
    if rank == 0:
        send = torch.zeros(16, dtype=torch.uint8)
        recv = torch.empty(16, dtype=torch.uint8)
        t0 = time.monotonic()
        try:
            comm.wait(comm.exchange(send, recv))
            q.put(("no-error", time.monotonic() - t0))
        except RuntimeError as e:
            q.put(("raised", time.monotonic() - t0, str(e)))
    else:
        time.sleep(6.0)  # the hung peer: never posts its send / recv
    os._exit(0)


def test_ring_wait_times_out_on_hung_peer():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get()
    for p in procs:
        p.join(timeout=30)
    assert res[0] == "raised", res
    assert 1.5 <= res[1] < 10.0, res
    assert "not complete" in res[2]

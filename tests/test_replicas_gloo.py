"""Multi-process (world_size 2, gloo on CPU) tests of the replica path:
the shared-memory JSQ / round-robin dispatcher assigns every request of a global trace
exactly once, JSQ steers load away from a slow replica, and the max-over-ranks /
sum-over-ranks aggregation bench.py uses reduces correctly."""
import os
import socket
import threading
import time

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, policy, service_s, n_req, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_21301_b200.dispatch import ReplicaBoard, Dispatcher, wait_assignment
    name = f"nova_test_board_{port}"
    if rank == 0:
        board = ReplicaBoard(name, world, n_req, create=True)
    dist.barrier()
    if rank != 0:
        board = ReplicaBoard(name, world, n_req, create=False)
    arrivals = [i * 0.004 for i in range(n_req)]
    t0 = time.monotonic() + 0.05
    mine, lat = [], []
    queue, lock = [], threading.Lock()
    state = {"submitted": 0, "done": 0, "stop": False}

    def server():                       # FIFO "front stage" with a fixed service time
        while not state["stop"] or queue:
            with lock:
                job = queue[0] if queue else None
            if job is None:
                time.sleep(0.0005)
                continue
            time.sleep(service_s[rank])
            with lock:
                queue.pop(0)
                state["done"] += 1
                lat.append(time.monotonic() - job)
                board.publish(rank, len(queue), state["submitted"])

    th = threading.Thread(target=server)
    th.start()
    disp = Dispatcher(board, arrivals, policy) if rank == 0 else None
    for i in range(n_req):
        while time.monotonic() < t0 + arrivals[i]:
            if disp:
                disp.assign_due(time.monotonic() - t0)
            time.sleep(0.0002)
        if disp:
            disp.assign_due(time.monotonic() - t0)
        r = wait_assignment(board, i)
        if r == rank:
            mine.append(i)
            with lock:
                queue.append(t0 + arrivals[i])
                state["submitted"] += 1
                board.publish(rank, len(queue), state["submitted"])
    state["stop"] = True
    th.join()
    # the aggregation bench.py performs: max latency over ranks, total requests over ranks
    t = torch.tensor([max(lat) if lat else 0.0], dtype=torch.float64)
    n = torch.tensor([float(len(mine))], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        out_q.put((gathered, t.item(), n.item(), max(lat) if lat else 0.0))
    dist.barrier()
    board.close()
    dist.destroy_process_group()


def _run(policy, service_s, n_req=60):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, policy, service_s, n_req, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


def test_jsq_assigns_exactly_once_and_balances():
    gathered, tmax, ntot, _ = _run("jsq", {0: 0.002, 1: 0.012})
    allreq = sorted(gathered[0] + gathered[1])
    assert allreq == list(range(60))                       # exactly once, nothing lost
    assert not set(gathered[0]) & set(gathered[1])
    assert len(gathered[0]) > len(gathered[1])             # the slow replica gets less work
    assert ntot == 60.0 and tmax > 0


def test_round_robin_control():
    gathered, _, ntot, _ = _run("rr", {0: 0.002, 1: 0.002}, n_req=20)
    assert gathered[0] == list(range(0, 20, 2)) and gathered[1] == list(range(1, 20, 2))
    assert ntot == 20.0

"""Replica request dispatcher (the paper's setting is one GPU (P:29,
P:155) and the path does not shard, so N GPUs run N independent engines behind a
host-side dispatcher; no collective on the data path).

Protocol (one node, one process per GPU): a board in POSIX shared memory holds, per
rank, the live front-stage backlog (requests submitted to that replica whose prefill
has not finished -- the quantity Eq. 5 calls N_pend) and the number of requests
the rank has submitted, plus, per request of the global trace, the rank it is assigned
to.  Rank 0 runs the dispatcher: at each arrival it computes each replica's load =
published backlog + requests assigned to it but not yet submitted, and assigns the
request to the least-loaded replica (join-shortest-queue; ties -> lowest rank) or
round-robin.  Every rank's submitter waits for the assignment slot of the next request
and submits it iff it is its own.  Each request is assigned exactly once, by one writer.
"""
from __future__ import annotations

import time
from multiprocessing import shared_memory

import numpy as np

UNASSIGNED = -1


class ReplicaBoard:
    """Shared-memory board: int64 backlog[world], int64 submitted[world], int32 assign[n]."""

    def __init__(self, name: str, world: int, n_requests: int, create: bool):
        self.world, self.n = world, n_requests
        size = 16 * world + 4 * max(1, n_requests)
        if create:
            try:
                old = shared_memory.SharedMemory(name=name)
                old.close()
                old.unlink()
            except FileNotFoundError:
                pass
            self.shm = shared_memory.SharedMemory(name=name, create=True, size=size)
        else:
            self.shm = None
            for _ in range(4000):
                try:
                    self.shm = shared_memory.SharedMemory(name=name)
                    break
                except FileNotFoundError:
                    time.sleep(0.005)
            if self.shm is None:
                raise RuntimeError(f"board {name} not found")
        self.backlog = np.ndarray((world,), dtype=np.int64, buffer=self.shm.buf, offset=0)
        self.submitted = np.ndarray((world,), dtype=np.int64, buffer=self.shm.buf, offset=8 * world)
        self.assign = np.ndarray((n_requests,), dtype=np.int32, buffer=self.shm.buf, offset=16 * world)
        if create:
            self.backlog[:] = 0
            self.submitted[:] = 0
            self.assign[:] = UNASSIGNED
        self.created = create

    def publish(self, rank: int, backlog: int, submitted: int) -> None:
        self.backlog[rank] = backlog
        self.submitted[rank] = submitted

    def close(self) -> None:
        del self.backlog, self.submitted, self.assign
        self.shm.close()
        if self.created:
            try:
                self.shm.unlink()
            except FileNotFoundError:
                pass


def choose(policy: str, load: np.ndarray, i: int) -> int:
    """JSQ on the front backlog (ties -> lowest rank) or round-robin."""
    if policy == "rr":
        return i % len(load)
    return int(np.argmin(load))     # argmin returns the first (lowest) index on ties


class Dispatcher:
    """Rank-0 dispatcher: `assign_due(now_s)` assigns every request whose arrival has passed."""

    def __init__(self, board: ReplicaBoard, arrivals_s, policy: str = "jsq"):
        self.board, self.arr, self.policy, self.next = board, list(arrivals_s), policy, 0
        self.assigned = np.zeros(board.world, dtype=np.int64)

    def loads(self) -> np.ndarray:
        return self.board.backlog.copy() + (self.assigned - self.board.submitted.copy())

    def assign_due(self, now_s: float) -> int:
        n = 0
        while self.next < len(self.arr) and self.arr[self.next] <= now_s:
            r = choose(self.policy, self.loads(), self.next)
            self.board.assign[self.next] = r
            self.assigned[r] += 1
            self.next += 1
            n += 1
        return n

    def done(self) -> bool:
        return self.next >= len(self.arr)


def wait_assignment(board: ReplicaBoard, i: int, timeout_s: float = 120.0) -> int:
    t0 = time.monotonic()
    while True:
        r = int(board.assign[i])
        if r != UNASSIGNED:
            return r
        if time.monotonic() - t0 > timeout_s:
            raise TimeoutError(f"request {i} never assigned")
        time.sleep(0.0001)

"""Test-only stand-in for an NCCL communicator on ONE GPU: every "rank" is a Python thread with
its own CUDA stream, and transfers are device copies on a side stream ordered purely by CUDA
events -- the semantics sharding.TorchComm relies on under NCCL (stream_ordered = True): a
transfer starts after both sides' streams reached the post (pack done), and wait() orders the
caller's stream after the transfer without blocking the host.  Lets the stream-ordered exchange
pipeline of sharding.py run on the single GPU gpurun provides (NCCL refuses two ranks on one
device)."""

import threading


class ThreadGroup:
    def __init__(self, world):
        import torch

        self.world = world
        self.cond = threading.Condition()
        self.box: dict = {}
        self.side = [torch.cuda.Stream() for _ in range(world)]

    def post(self, key, value):
        with self.cond:
            self.box.setdefault(key, []).append(value)
            self.cond.notify_all()

    def take(self, key, timeout=120.0):
        with self.cond:
            ok = self.cond.wait_for(lambda: self.box.get(key), timeout=timeout)
            if not ok:
                raise TimeoutError(f"no message for {key}")
            return self.box[key].pop(0)


class _Work:
    def __init__(self, events):
        self.events = events

    def wait(self):
        import torch

        s = torch.cuda.current_stream()
        for e in self.events:
            s.wait_event(e)


class ThreadComm:
    CHUNK_BYTES = 1 << 15
    stream_ordered = True

    def __init__(self, group: ThreadGroup, rank: int):
        self.g = group
        self.rank = rank
        self.world = group.world
        self.seq: dict = {}

    def owns(self, shard_id, owner):
        return owner[shard_id] == self.rank

    def _tag(self, peer):
        k = self.seq.get(peer, 0)
        self.seq[peer] = k + 1
        return k

    def ialltoall(self, triples):
        import torch

        posted = torch.cuda.Event()
        posted.record()  # after this rank's packs on its current stream
        tags = []
        for send, recv, peer in triples:
            t = self._tag(peer)
            tags.append(t)
            self.g.post(("data", self.rank, peer, t), (send, posted))
        side = self.g.side[self.rank]
        works = []
        for (send, recv, peer), t in zip(triples, tags):
            psend, pev = self.g.take(("data", peer, self.rank, t))
            side.wait_event(pev)
            side.wait_event(posted)  # my receive buffer is free once my stream got here
            with torch.cuda.stream(side):
                recv.copy_(psend)
            done = torch.cuda.Event()
            done.record(side)
            # the peer may reuse its send buffer only after my copy read it
            self.g.post(("done", self.rank, peer, t), done)
            works.append(done)
        for (_, _, peer), t in zip(triples, tags):
            works.append(self.g.take(("done", peer, self.rank, t)))
        return [_Work(works)]

    def isendrecv(self, send, recv, peer):
        return self.ialltoall([(send, recv, peer)])

    def all_gather(self, t):
        import torch

        torch.cuda.current_stream().synchronize()
        k = self._tag(-1)
        for r in range(self.world):
            self.g.post(("ag", self.rank, r, k), t.clone())
        torch.cuda.current_stream().synchronize()
        return [self.g.take(("ag", r, self.rank, k)) for r in range(self.world)]

    def barrier(self):
        self.all_gather(__import__("torch").zeros(1, device="cuda"))


def run_ranks(world, fn):
    """fn(comm) on `world` threads, each with its own current CUDA stream; returns the results
    in rank order (re-raises the first failure)."""
    import torch

    group = ThreadGroup(world)
    out = [None] * world
    err = []

    def body(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(ThreadComm(group, r))
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            with group.cond:
                group.cond.notify_all()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out

"""Rank-to-rank exchange of the spatially partitioned transform and solve
(DESIGN.md section 6).

A level grid of L rows is split into `world` contiguous row strips
(`partition.row_strips`); rank r owns strip r of every distributed level.
Level operators are row-major with a fixed number of elements per grid row
(box rows of a grid row are contiguous), so everything a rank needs from the
others is a set of whole grid rows:

  halo(buf, L, row_elems, up, down)      rows [r0-up, r0) and [r1, r1+down)
                                         filled from their owners
  halo_add(buf, L, row_elems, up, down)  the reverse: contributions a rank
                                         computed for rows it does not own are
                                         added into the owner's rows
  allreduce(t, op)                       sum / max / min of small tensors
  allgather_rows(buf, L, row_elems)      every rank ends with all rows

Two transports implement them with the same semantics:

  TorchComm   one process per GPU over torch.distributed -- NCCL send/recv
              and all-reduce on device buffers (NVLink / NVSwitch); with the
              gloo backend the rows are staged through host memory (the
              2-process tests: CPU tensors, or two ranks sharing one GPU).
  ThreadComm  `world` ranks as threads of one process, each with its own
              CUDA stream, exchanging by device copies ordered with events:
              the single-GPU parity transport (NCCL cannot place two ranks
              on one device).  No kernel ever waits on another rank's kernel;
              ordering is host barriers plus stream events.
"""

from __future__ import annotations

import threading

import torch

from .partition import row_strips

__all__ = ["Comm", "SelfComm", "TorchComm", "ThreadComm", "run_threads"]


def _overlap(a0, a1, b0, b1):
    lo, hi = max(a0, b0), min(a1, b1)
    return (lo, hi) if hi > lo else None


class Comm:
    """Base: strip geometry and the row bookkeeping shared by the transports."""

    world = 1
    rank = 0

    def strip(self, L):
        """This rank's rows [r0, r1) of an L-row grid."""
        return row_strips(L, self.world)[self.rank]

    def _wanted(self, L, up, down, rank):
        """Row ranges rank `rank` wants from the others: [(peer, a, b)]."""
        strips = row_strips(L, self.world)
        r0, r1 = strips[rank]
        out = []
        for lo, hi in ((max(r0 - up, 0), r0), (r1, min(r1 + down, L))):
            if hi <= lo:
                continue
            for peer, (p0, p1) in enumerate(strips):
                if peer == rank:
                    continue
                ov = _overlap(lo, hi, p0, p1)
                if ov:
                    out.append((peer, ov[0], ov[1]))
        return out

    # single rank: nothing to exchange
    def halo(self, buf, L, row_elems, up, down):
        return

    def halo_add(self, buf, L, row_elems, up, down):
        return

    def halo_many(self, items):
        """Several halos [(buf, L, row_elems, up, down)] as one exchange."""
        for it in items:
            self.halo(*it)

    def allreduce(self, t, op="sum"):
        return t

    def allgather_rows(self, buf, L, row_elems):
        return

    def broadcast(self, t, src):
        """t of rank `src` on every rank."""
        return t

    def barrier(self):
        return


class SelfComm(Comm):
    """world = 1."""


_OPS = {"sum": "SUM", "max": "MAX", "min": "MIN"}


class TorchComm(Comm):
    """torch.distributed transport (NCCL on GPUs; gloo stages through the host)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        self.bytes_sent = 0

    def _stage(self, t):
        return self.backend == "gloo" and t.is_cuda

    def _exchange(self, buf, sends, recvs, row_elems, add=False):
        """sends / recvs: [(peer, a, b)] row ranges of buf."""
        self._exchange_many([(buf, sends, recvs, row_elems)], add)

    def _exchange_many(self, jobs, add=False):
        """jobs: [(buf, sends, recvs, row_elems)] -- one batch of P2P ops (one
        NCCL group): the order of the jobs is the same on every rank, so the
        messages of a pair of ranks match in order."""
        dist = self.dist
        ops, landing, keep = [], [], []
        for buf, sends, recvs, row_elems in jobs:
            for peer, a, b in recvs:
                view = buf[a * row_elems:b * row_elems]
                if add or self._stage(buf):
                    tmp = torch.empty(view.shape, dtype=buf.dtype,
                                      device="cpu" if self._stage(buf) else buf.device)
                    landing.append((view, tmp))
                    ops.append(dist.P2POp(dist.irecv, tmp, peer, self.group))
                else:
                    ops.append(dist.P2POp(dist.irecv, view, peer, self.group))
            for peer, a, b in sends:
                view = buf[a * row_elems:b * row_elems]
                if self._stage(buf):
                    view = view.cpu()
                    keep.append(view)
                self.bytes_sent += view.numel() * view.element_size()
                ops.append(dist.P2POp(dist.isend, view, peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for view, tmp in landing:  # fixed order: ascending source rows
            src = tmp.to(view.device, non_blocking=False)
            if add:
                view.add_(src)
            else:
                view.copy_(src)

    def _halo_job(self, buf, L, row_elems, up, down):
        recvs = self._wanted(L, up, down, self.rank)
        sends = [(peer, a, b) for peer in range(self.world) if peer != self.rank
                 for (src, a, b) in self._wanted(L, up, down, peer) if src == self.rank]
        return (buf, sends, recvs, row_elems)

    def halo(self, buf, L, row_elems, up, down):
        if self.world == 1 or (up <= 0 and down <= 0):
            return
        self._exchange_many([self._halo_job(buf, L, row_elems, up, down)])

    def halo_many(self, items):
        if self.world == 1:
            return
        jobs = [self._halo_job(*it) for it in items if it[3] > 0 or it[4] > 0]
        if jobs:
            self._exchange_many(jobs)

    def halo_add(self, buf, L, row_elems, up, down):
        if self.world == 1 or (up <= 0 and down <= 0):
            return
        # what I hold for others = the rows I would want in a halo() of the
        # same widths; what I receive = contributions to my own rows
        sends = self._wanted(L, up, down, self.rank)
        recvs = [(peer, a, b) for peer in range(self.world) if peer != self.rank
                 for (src, a, b) in self._wanted(L, up, down, peer) if src == self.rank]
        self._exchange(buf, sends, sorted(recvs), row_elems, add=True)

    def allreduce(self, t, op="sum"):
        if self.world == 1:
            return t
        rop = getattr(self.dist.ReduceOp, _OPS[op])
        if self._stage(t):
            h = t.cpu()
            self.dist.all_reduce(h, op=rop, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=rop, group=self.group)
        return t

    def allgather_rows(self, buf, L, row_elems):
        if self.world == 1:
            return
        for r, (a, b) in enumerate(row_strips(L, self.world)):
            if b <= a:
                continue
            view = buf[a * row_elems:b * row_elems]
            if self._stage(buf):
                h = view.cpu()
                self.dist.broadcast(h, src=self._global(r), group=self.group)
                if r != self.rank:
                    view.copy_(h)
            else:
                self.dist.broadcast(view, src=self._global(r), group=self.group)
            if r == self.rank:
                self.bytes_sent += view.numel() * view.element_size()

    def broadcast(self, t, src):
        if self.world == 1:
            return t
        if self._stage(t):
            h = t.cpu()
            self.dist.broadcast(h, src=self._global(src), group=self.group)
            if src != self.rank:
                t.copy_(h)
        else:
            self.dist.broadcast(t, src=self._global(src), group=self.group)
        if src == self.rank:
            self.bytes_sent += t.numel() * t.element_size()
        return t

    def _global(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)


class _Hub:
    """Shared state of the in-process ranks."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slot = [None] * world
        self.done = [None] * world
        self.error = None


class ThreadComm(Comm):
    """`world` ranks as threads of one process sharing one GPU (or CPU
    tensors): rows move by tensor copies on the receiving rank's stream,
    ordered after the owner's work by an event, and the owner's stream waits
    for its readers before it continues."""

    def __init__(self, hub, rank):
        self.hub = hub
        self.world = hub.world
        self.rank = rank
        self.bytes_sent = 0

    @staticmethod
    def _event(t):
        if not t.is_cuda:
            return None
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(t.device))
        return ev

    @staticmethod
    def _wait(t, ev):
        if ev is not None:
            torch.cuda.current_stream(t.device).wait_event(ev)

    def _sync(self):
        try:
            self.hub.bar.wait()
        except threading.BrokenBarrierError:
            raise RuntimeError("another in-process rank failed") from self.hub.error

    def _publish(self, buf):
        self.hub.slot[self.rank] = (buf, self._event(buf))
        self._sync()

    def _retire(self, buf):
        """After reading the peers' buffers: let every owner wait for its readers."""
        self.hub.done[self.rank] = self._event(buf)
        self._sync()
        for r in range(self.world):
            if r != self.rank:
                self._wait(buf, self.hub.done[r])
        self._sync()

    def halo(self, buf, L, row_elems, up, down):
        if self.world == 1 or (up <= 0 and down <= 0):
            return
        self._publish(buf)
        for peer, a, b in self._wanted(L, up, down, self.rank):
            src, ev = self.hub.slot[peer]
            self._wait(buf, ev)
            buf[a * row_elems:b * row_elems].copy_(src[a * row_elems:b * row_elems])
            self.bytes_sent += (b - a) * row_elems * buf.element_size()
        self._retire(buf)

    def halo_add(self, buf, L, row_elems, up, down):
        if self.world == 1 or (up <= 0 and down <= 0):
            return
        self._publish(buf)
        # contributions the peers hold for my rows, added in ascending peer order
        tmp = []
        for peer in range(self.world):
            if peer == self.rank:
                continue
            for src_rank, a, b in self._wanted(L, up, down, peer):
                if src_rank != self.rank:
                    continue
                src, ev = self.hub.slot[peer]
                self._wait(buf, ev)
                tmp.append((a, b, src[a * row_elems:b * row_elems].clone()))
        self._retire(buf)
        for a, b, t in tmp:
            buf[a * row_elems:b * row_elems].add_(t)

    def allreduce(self, t, op="sum"):
        if self.world == 1:
            return t
        self._publish(t)
        acc = None
        for r in range(self.world):  # fixed rank order on every rank
            src, ev = self.hub.slot[r]
            self._wait(t, ev)
            if acc is None:
                acc = src.clone()
            elif op == "sum":
                acc += src
            elif op == "max":
                acc = torch.maximum(acc, src)
            else:
                acc = torch.minimum(acc, src)
        self._retire(t)
        t.copy_(acc)
        return t

    def allgather_rows(self, buf, L, row_elems):
        if self.world == 1:
            return
        self._publish(buf)
        for peer, (a, b) in enumerate(row_strips(L, self.world)):
            if peer == self.rank or b <= a:
                continue
            src, ev = self.hub.slot[peer]
            self._wait(buf, ev)
            buf[a * row_elems:b * row_elems].copy_(src[a * row_elems:b * row_elems])
        self._retire(buf)

    def broadcast(self, t, src):
        if self.world == 1:
            return t
        self._publish(t)
        if src != self.rank:
            buf, ev = self.hub.slot[src]
            self._wait(t, ev)
            t.copy_(buf)
        self._retire(t)
        return t

    def barrier(self):
        self._sync()


def run_threads(world, fn, *args, device=None):
    """Run fn(comm, *args) on `world` in-process ranks (threads, one CUDA
    stream each); returns the list of results in rank order.  The first
    exception of any rank is re-raised."""
    hub = _Hub(world)
    out, errs = [None] * world, [None] * world

    def body(r):
        try:
            comm = ThreadComm(hub, r)
            if device is not None and torch.cuda.is_available():
                torch.cuda.set_device(device)
                with torch.cuda.stream(torch.cuda.Stream(device=device)):
                    out[r] = fn(comm, *args)
                    torch.cuda.current_stream().synchronize()
            else:
                out[r] = fn(comm, *args)
        except BaseException as e:  # noqa: BLE001 -- re-raised on the caller
            errs[r] = e
            hub.error = hub.error or e
            hub.bar.abort()

    ts = [threading.Thread(target=body, args=(r,), name=f"gb-rank{r}") for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, RuntimeError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    return out

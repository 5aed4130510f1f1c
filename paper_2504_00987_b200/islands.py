"""Island model over the GPUs of one node (one process per GPU).

Each rank owns an independent device-resident replica set (labs_solver; global
replica ids rank*R + r, seeds base_seed + id — the reference's seeding rule,
proj/src/parallel.cpp:38). Ranks never share a data path: between device
epochs they exchange only
  * the stop decision and the best key (E << 32 | global replica) —
    all_reduce(MIN) over a packed int64 (SharedState::publish's "strictly
    lower energy wins" becomes "lowest key wins"; parallel.cpp:10-15), and
  * optionally k elites per rank (all_gather over NCCL/NVLink, k x (words + E)
    — a few hundred bytes), offered to every replica's population.
The reference has no migration; with exchange_every == 0 the
island run is exactly R*world independent reference replicas.

The collective plumbing is torch.distributed (NCCL on GPUs, gloo in the CPU
tests); the solver is any object with the labs_solver surface of
paper_2504_00987_b200.capi.Solver.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch
import torch.distributed as dist


def pack_key(energy: int, replica: int) -> int:
    return (int(energy) << 32) | (int(replica) & 0xFFFFFFFF)


def unpack_key(key: int):
    return key >> 32, key & 0xFFFFFFFF


@dataclass
class IslandReport:
    epochs: int = 0
    exchanges: int = 0
    best_energy: int = -1
    best_replica: int = -1
    reached: bool = False
    seconds: float = 0.0
    history: list = field(default_factory=list)


class Islands:
    """Drive one rank's solver through epochs with cross-rank coordination.

    Device-side stop: with link_stops=True (CUDA solvers, world > 1) every
    rank exports its solver's stop flag through CUDA IPC and raises the
    others' flags from the kernel the moment one of its replicas reaches the
    target (labs_solver_set_peer_stops), so a stop crosses GPUs over NVLink
    within one memetic iteration instead of waiting for the epoch's host
    all_reduce. The per-epoch all_reduce remains for the best key and for
    termination."""

    def __init__(self, solver, n: int, k_elites: int = 16, device=None, group=None,
                 link_stops: bool = True):
        self.solver, self.n, self.k = solver, n, k_elites
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device if device is not None else torch.device("cpu")
        # gloo moves host tensors only: stage device buffers through the host
        backend = dist.get_backend(group) if dist.is_initialized() else None
        self.stage = self.device.type == "cuda" and backend == "gloo"
        self.comm_device = torch.device("cpu") if self.stage else self.device
        nw = (n + 63) // 64
        self.el_w = torch.zeros(k_elites * nw, dtype=torch.int64, device=self.device)
        self.el_e = torch.zeros(k_elites, dtype=torch.int64, device=self.device)
        self.all_w = torch.zeros(self.world * k_elites * nw, dtype=torch.int64, device=self.device)
        self.all_e = torch.zeros(self.world * k_elites, dtype=torch.int64, device=self.device)
        self.peer_ptrs = []
        if link_stops and self.world > 1 and hasattr(solver, "stop_flag"):
            self._link_stops()

    def _link_stops(self):
        ctx = self.solver.ctx
        mine = ctx.ipc_export(self.solver.stop_flag)
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=self.group)
        self.peer_ptrs = [ctx.ipc_open(h) for r, h in enumerate(handles) if r != self.rank]
        self.solver.set_peer_stops(self.peer_ptrs)
        dist.barrier(group=self.group)  # every flag mapped before any kernel runs

    def close(self):
        """Unlink and unmap the peers' stop flags (before the solver goes)."""
        if self.peer_ptrs:
            self.solver.set_peer_stops([])
            self.solver.sync()
            if self.world > 1:
                dist.barrier(group=self.group)  # no peer still raising our flag
            for p in self.peer_ptrs:
                self.solver.ctx.ipc_close(p)
            self.peer_ptrs = []
            if self.world > 1:
                dist.barrier(group=self.group)  # every mapping closed before any flag is freed

    def _allreduce(self, values, op):
        t = torch.tensor(values, dtype=torch.int64, device=self.comm_device)
        if self.world > 1:
            dist.all_reduce(t, op=op, group=self.group)
        return t.tolist()

    def exchange(self, rotation: int):
        """Export top-k, all_gather across ranks, offer to every replica."""
        self.solver.export_elites(self.k, self.el_w.data_ptr(), self.el_e.data_ptr())
        self.solver.sync()  # the export (solver stream) is complete
        if self.world > 1:
            src_w = self.el_w.cpu() if self.stage else self.el_w
            src_e = self.el_e.cpu() if self.stage else self.el_e
            dst_w = torch.empty(self.all_w.shape, dtype=torch.int64, device=self.comm_device)
            dst_e = torch.empty(self.all_e.shape, dtype=torch.int64, device=self.comm_device)
            dist.all_gather_into_tensor(dst_w, src_w, group=self.group)
            dist.all_gather_into_tensor(dst_e, src_e, group=self.group)
            self.all_w.copy_(dst_w)
            self.all_e.copy_(dst_e)
        else:
            self.all_w.copy_(self.el_w)
            self.all_e.copy_(self.el_e)
        # The gather and copies ran on torch's stream; the import runs on the
        # solver's own stream, so it must not start before they finish.
        if self.device.type == "cuda":
            torch.cuda.current_stream(self.device).synchronize()
        self.solver.import_elites(self.world * self.k, self.all_w.data_ptr(),
                                  self.all_e.data_ptr(), rotation=rotation)

    def global_best(self):
        st = self.solver.status()
        key = pack_key(st["best_energy"], st["best_replica"]) if st["best_replica"] >= 0 \
            else (1 << 62)
        running = st["running"]
        key, = self._allreduce([key], dist.ReduceOp.MIN)
        running, = self._allreduce([running], dist.ReduceOp.SUM)
        return key, running

    def run(self, target: int, epoch_seconds: float, exchange_every: int = 0,
            max_seconds: float | None = None) -> IslandReport:
        """Epochs until some replica on some rank reaches `target`, every
        replica finished, or max_seconds elapsed (same wall on all ranks: the
        decision is all-reduced)."""
        rep = IslandReport()
        t0 = time.perf_counter()
        while True:
            self.solver.run(epoch_seconds=epoch_seconds, race=True)
            rep.epochs += 1
            if exchange_every and rep.epochs % exchange_every == 0:
                self.exchange(rotation=rep.epochs)
                rep.exchanges += 1
            key, running = self.global_best()
            e, r = unpack_key(key)
            rep.history.append(e)
            timed_out = max_seconds is not None and time.perf_counter() - t0 >= max_seconds
            stop_flags, = self._allreduce([1 if timed_out else 0], dist.ReduceOp.MAX)
            if e <= target or running == 0 or stop_flags:
                if e <= target or stop_flags:
                    self.solver.request_stop()
                rep.best_energy, rep.best_replica = e, r
                rep.reached = e <= target
                break
        rep.seconds = time.perf_counter() - t0
        return rep

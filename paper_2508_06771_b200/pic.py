"""NEXT f2: the subcycled kinetic loop around the collision operator.

Table 2 of the paper splits a PIC time step into S1 (DSMC-Coul,
this library's ``coulomb_collide``), S2a (electron-heavy collisions, out of
scope: LXCat data), S2b/S2c (field interpolation and push) and the P2C/PDE
steps S3/S4.  Production runs take "ten DSMC-Coll / recombination / Coulombic
steps per PDE solve" (subcycling; "multiple collision kernels are
performed for each time step of the continuum physics").  ``PicLoop`` runs
that loop restricted to the path:

  per substep   S1   coulomb_collide: bins the pushed particles (nearly sorted:
                     the previous output order), pairs, collides; its
                     per-cell moments are the P2C of the post-collision state
                S2b+S2c the push: v += dt (q/m) E[cell], x += dt v, boundary, new
                     cell id — a separate cc_push reading the positions through
                     perm_out (the default, fused=False: measured faster at C4,
                     DESIGN §6) or fused into the collision call's output stage
                     (cc_params.push, fused=True); same bits
  per field step     (every ``subcycles`` substeps) the lagged per-cell Coulomb
                     logarithm from the last moments (R21, cc_coulomb_log), fed to
                     the next substeps as ln_lambda_arr; E is held fixed (the PDE
                     solves S4 are outside the paper's own scope).

One GPU: the whole field step (``subcycles`` x 13 kernel launches) is captured
once into a CUDA graph and replayed; the random streams advance through a
device step counter (cc_params.step_dev: effective step = substep index +
subcycles x field-step index), so graph replay and eager execution give
bit-identical results.  Several GPUs (cell-range shards, ``dist``): eager, with
a device-side migration (``dist.Migrator``: fixed-capacity slots, positions as
payload, no host synchronisation) after each push; the particle buffers have a
fixed number of dead-padded slots (``capacity``) and are allocated once.

All per-particle arithmetic runs in the library's CUDA kernels; this module
only sequences calls and owns buffers.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import coulomb as cc
from .coulomb import M_E, Q_E, Grid


class PicLoop:
    def __init__(self, x: torch.Tensor, v: torch.Tensor, cell: torch.Tensor, grid: Grid, *, dt: float,
                 weight: float, cell_volume: float, E: Optional[torch.Tensor] = None,
                 q_over_m: float = -Q_E / M_E, seed: int = 42, subcycles: int = 10, ln_lambda: float = 10.0,
                 coulomb_log_feedback: bool = True, graph: bool = True, flags: int = 0,
                 dist_ops=None, group=None, cell_base: int = 0, cells: Optional[int] = None, fused: bool = False,
                 capacity: Optional[int] = None, mig_cap: Optional[int] = None):
        if subcycles < 1 or subcycles % 2:
            raise ValueError("subcycles must be a positive even number (ping-pong buffers)")
        self.dev = cell.device
        self.grid, self.dt, self.E, self.qm = grid, dt, E, q_over_m
        self.seed, self.k, self.flags = seed, subcycles, flags
        self.weight, self.volume = weight, cell_volume
        self.feedback = coulomb_log_feedback
        self.dist_ops, self.group = dist_ops, group
        self.cell_base = cell_base
        self.cells = grid.cells if cells is None else cells
        self.use_graph = graph and dist_ops is None
        self.fused = fused            # push inside the collision call's output stage (cc_params.push)
        self.field_steps = 0
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.lnl = torch.full((self.cells,), float(ln_lambda), dtype=torch.float64, device=self.dev)
        self.moments = torch.zeros((self.cells, cc.CC_MOMENTS_LEN), dtype=torch.float64, device=self.dev)
        self.diag = torch.zeros(cc.CC_DIAG_LEN, dtype=torch.float64, device=self.dev)
        n0 = cell.numel()
        if dist_ops is not None and capacity is None:
            capacity = n0 + n0 // 4 + 1024          # room for arrivals (dead-padded slots)
        self._alloc(x, v, cell, capacity)
        self._graph = None
        self.migrator = None
        if dist_ops is not None:
            import torch.distributed as tdist
            from . import dist as ccd
            world = tdist.get_world_size(group) if tdist.is_initialized() else 1
            rank = tdist.get_rank(group) if tdist.is_initialized() else 0
            bounds = ccd.owner_bounds(grid.cells, world)
            self.migrator = ccd.Migrator(self.n, bounds, rank, mig_cap or max(1024, n0 // 20), self.dev,
                                         xrows=grid.dims, comm=dist_ops.nccl,
                                         exchange=None if dist_ops.nccl is not None else ccd.torch_exchange(group))

    # ------------------------------------------------------------------ buffers
    def _alloc(self, x, v, cell, capacity=None):
        n0 = cell.numel()
        n = max(n0, capacity or n0)
        self.n = n
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.x = [torch.zeros((3, n), **f64), torch.zeros((3, n), **f64)]   # rows >= dims never written by cc_push
        self.v = [torch.zeros((3, n), **f64), torch.empty((3, n), **f64)]
        self.cell = [torch.full((n,), -1, dtype=torch.int32, device=self.dev),
                     torch.empty(n, dtype=torch.int32, device=self.dev)]
        self.x[0][:, :n0].copy_(x)
        self.v[0][:, :n0].copy_(v)
        self.cell[0][:n0].copy_(cell)                     # slots beyond n0: dead padding
        self.perm = torch.empty(n, dtype=torch.int32, device=self.dev)
        self.ws = cc.alloc_workspace(n, self.cells, self.dev)
        self.a = 0

    @property
    def state(self):
        """(x [3][n], v [3][n], cell [n] local ids, -1 dead) after the last substep."""
        return self.x[self.a], self.v[self.a], self.cell[self.a]

    # ------------------------------------------------------------------ one substep
    def _substep(self, s: int):
        a, b = self.a, self.a ^ 1
        out = cc.CollideOut(self.v[b], self.cell[b], self.perm, self.moments, self.diag)
        push = None
        if self.fused:
            push = dict(grid=self.grid, x_in=self.x[a], x_out=self.x[b], E=self.E, q_over_m=self.qm)
        cc.coulomb_collide(self.v[a], self.cell[a], self.cells, dt=self.dt, weight=self.weight,
                           cell_volume=self.volume, ln_lambda_arr=self.lnl, cell_base=self.cell_base,
                           seed=self.seed, step=s, out=out, workspace=self.ws, flags=self.flags,
                           step_dev=self.step_dev, push=push)
        if not self.fused:
            cc.cc_push(self.x[a], self.v[b], self.cell[b], self.grid, dt=self.dt, q_over_m=self.qm, E=self.E,
                       perm=self.perm, x_out=self.x[b], cells=self.cells, cell_base=self.cell_base)
        self.a = b

    def _field_step_body(self):
        for s in range(self.k):
            self._substep(s)
        if self.feedback:
            lnl = cc.cc_coulomb_log(self.moments)
            self.lnl.copy_(lnl)
        cc.cc_step_advance(self.step_dev, self.k)

    # ------------------------------------------------------------------ public
    def field_step(self):
        """``subcycles`` substeps (S1 + S2b/S2c each) and the field-step feedback."""
        if self.dist_ops is not None:
            self._field_step_dist()
        elif not self.use_graph:
            self._field_step_body()
        else:
            if self._graph is None:
                # warm-up outside capture (lazy library state, allocator), then capture
                a0 = self.a
                saved = [t.clone() for t in (self.x[a0], self.v[a0], self.cell[a0], self.lnl, self.step_dev)]
                side = torch.cuda.Stream(self.dev)
                side.wait_stream(torch.cuda.current_stream(self.dev))
                with torch.cuda.stream(side):
                    self._field_step_body()
                torch.cuda.current_stream(self.dev).wait_stream(side)
                self.a = a0
                for t, sv in zip((self.x[a0], self.v[a0], self.cell[a0], self.lnl, self.step_dev), saved):
                    t.copy_(sv)
                self._graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self._graph):
                    self._field_step_body()
                self.a = a0
            self._graph.replay()
        self.field_steps += 1

    def _field_step_dist(self):
        for s in range(self.k):
            self._substep(s)
            # device-side migration in the fixed slots (no host sync, no re-allocation):
            # leavers out, GLOBAL -> LOCAL ids, arrivals into the dead tail [L, n)
            self.migrator(self.v[self.a], self.x[self.a], self.cell[self.a], self.diag)
        if self.feedback:
            self.lnl.copy_(cc.cc_coulomb_log(self.moments))
        cc.cc_step_advance(self.step_dev, self.k)

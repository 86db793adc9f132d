"""Lagrangian particle tracking (Algorithm 1, §6.7; SPEC.md:458-477
`run_particles`).

One step of Algorithm 1 on the device:
  Interpolate  u at the particles from their current records (fpx_findpts_eval)
  ParticleRHS  a = (u - v) / tau                     } one fused kernel,
  Integrate    2nd-order Adams-Bashforth for (x, v)  } fpx_particles_advance
  ParticleBC   periodic wrap of the box              }
  Find         records at the new positions (fpx_find; routed over ranks)
  (removal)    particles NOT_FOUND after the wrap are dropped and counted
  Migrate      when the global fraction of rank-non-local particles > 0.1,
               every particle moves to the rank that owns its element
               (one all-to-all of the particle state).
The fluid solve (FluidSolve) is out of scope: the velocity is a given field.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field as dfield

import torch

from . import _C, engine, transport
from .invmap import NOT_FOUND

__all__ = ["ParticleState", "init_particles", "advance", "run_particles", "MIGRATE_FRACTION"]

MIGRATE_FRACTION = 0.1  # Algorithm 1: migrate when the non-local fraction exceeds this


@dataclass
class ParticleState:
    """x, v [n, d] on the device; f_prev = (v_prev, a_prev) of the previous step
    for Adams-Bashforth; `records` of the current positions."""

    x: torch.Tensor
    v: torch.Tensor
    tau: float
    v_prev: torch.Tensor | None = None
    a_prev: torch.Tensor | None = None
    records: engine.FindRecords | None = None
    step: int = 0
    removed: int = 0
    migrations: int = 0
    timings: dict = dfield(default_factory=dict)
    # per step: (global non-local fraction after the find, migrated?)
    history: list = dfield(default_factory=list)

    def __len__(self) -> int:
        return int(self.x.shape[0])


def init_particles(S: engine.EngineSetup, x, v=None, tau: float = 5.0) -> ParticleState:
    """Particles at x (velocity v, default 0) with their first records."""
    xt = torch.as_tensor(x, dtype=torch.float64).to(S.device).contiguous()
    vt = torch.zeros_like(xt) if v is None else \
        torch.as_tensor(v, dtype=torch.float64).to(S.device).contiguous()
    if tau <= 0:
        raise ValueError("tau must be > 0")
    st = ParticleState(xt, vt, float(tau), torch.zeros_like(xt), torch.zeros_like(xt))
    st.records = engine.find(S, st.x)
    _drop_not_found(st)
    return st


def _drop_not_found(st: ParticleState) -> None:
    keep = st.records.code != NOT_FOUND
    lost = int(keep.numel() - keep.sum())
    if lost:
        st.removed += lost
        st.x, st.v = st.x[keep].contiguous(), st.v[keep].contiguous()
        st.v_prev, st.a_prev = st.v_prev[keep].contiguous(), st.a_prev[keep].contiguous()
        r = st.records
        st.records = engine.FindRecords(r.code[keep], r.rank[keep], r.elem[keep], r.r[keep],
                                        r.dist[keep], None, r.stats)


def _migrate(S: engine.EngineSetup, st: ParticleState) -> None:
    """Send every particle to the rank that owns its element (one exchange of
    x | v | v_prev | a_prev), then find the arrivals locally."""
    G = S.group
    rows = torch.cat([st.x, st.v, st.v_prev, st.a_prev], dim=1)
    dest = st.records.rank.long()
    order = torch.argsort(dest, stable=True)   # rows grouped by owner rank
    recv, _ = transport.exchange_packed(G, rows[order], torch.bincount(dest, minlength=G.size))
    d = st.x.shape[1]
    st.x, st.v = recv[:, :d].contiguous(), recv[:, d:2 * d].contiguous()
    st.v_prev, st.a_prev = recv[:, 2 * d:3 * d].contiguous(), recv[:, 3 * d:].contiguous()
    st.records = engine.find(S, st.x)
    st.migrations += 1


def nonlocal_fraction(S: engine.EngineSetup, st: ParticleState) -> float:
    """Global fraction of particles whose owning rank is not the holding rank."""
    G = S.group
    if G.single:
        return 0.0
    loc = int((st.records.rank != G.rank).sum())
    tot = transport.allgather_counts(G, len(st))
    nl = transport.allgather_counts(G, loc)
    return sum(nl) / max(1, sum(tot))


def advance(S: engine.EngineSetup, velocity, st: ParticleState, dt: float, box=None,
            periodic: int = 0b111) -> ParticleState:
    """One step of Algorithm 1 (see the module docstring).  `box` = (lo, hi)
    of the periodic domain; bit c of `periodic` wraps axis c."""
    d = S.phys_dim
    L = _C.lib()
    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for k in ("interpolate", "integrate", "find")}
    ev["interpolate"][0].record()
    u = engine.interpolate(S, velocity, st.records)
    ev["interpolate"][1].record()
    if u.shape[1] != d:
        raise ValueError(f"velocity field has {u.shape[1]} components, need {d}")
    u = u.contiguous()
    boxa = None
    if periodic:
        if box is None:
            raise ValueError("periodic wrapping needs the box (lo, hi)")
        boxa = (torch.tensor([*box[0], *box[1]], dtype=torch.float64)).contiguous()
    ev["integrate"][0].record()
    _C.check(L.fpx_particles_advance(d, len(st), _C.ptr(st.x), _C.ptr(st.v), _C.ptr(u),
                                     _C.ptr(st.v_prev), _C.ptr(st.a_prev), st.tau, float(dt),
                                     1 if st.step == 0 else 0,
                                     boxa.data_ptr() if boxa is not None else None,
                                     int(periodic) if boxa is not None else 0,
                                     _C.stream_handle()), "fpx_particles_advance")
    ev["integrate"][1].record()
    ev["find"][0].record()
    # re-location starts on each particle's previous element (hinted find:
    # no prefilter; the records are those of a find without hint)
    hint = st.records.elem if S.group.single and len(st) else None
    st.records = engine.find(S, st.x, hint=hint)
    ev["find"][1].record()
    _drop_not_found(st)
    frac = nonlocal_fraction(S, st)
    migrate = frac > MIGRATE_FRACTION
    if migrate:
        _migrate(S, st)
    st.history.append((frac, migrate))
    st.step += 1
    torch.cuda.synchronize()
    for k, (a, b) in ev.items():
        st.timings[k] = st.timings.get(k, 0.0) + a.elapsed_time(b)
    return st


def run_particles(S: engine.EngineSetup, velocity, x, v=None, tau: float = 5.0,
                  dt: float = 1e-3, steps: int = 100, box=None, periodic: int = 0b111) -> dict:
    """SPEC.md:466 run_particles: `steps` steps of Algorithm 1 from positions
    x.  Returns the trajectory summary (final state, counts, per-phase ms)."""
    t0 = time.perf_counter()
    velocity = engine._field_of(S, velocity)  # upload once
    st = init_particles(S, x, v, tau)
    n0 = len(st) + st.removed
    for _ in range(steps):
        advance(S, velocity, st, dt, box, periodic)
    return {"state": st, "particles": len(st), "initial": n0, "removed": st.removed,
            "migrations": st.migrations, "steps": steps, "phase_ms": dict(st.timings),
            "wall_s": time.perf_counter() - t0}

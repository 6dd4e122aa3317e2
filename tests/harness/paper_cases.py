"""The paper's benchmark scenarios as input recipes (reference
scenarios.py:20-156, restated as a table of cases + one assembly routine).

Test harness only: these build (ScenarioSpec, FlowState) pairs that the
acceptance, sweep and p > 1 tests hand to the GPU path.
"""

from __future__ import annotations

import numpy as np

from paper_2505_17025_b200.bathymetry import (GRAVITY, FlatBottom, HammackPlate, SlideMotion,
                                              WhittakerSlide, hammack_time_constant)
from paper_2505_17025_b200.grid import FlowState, GridSpec, NodalField
from paper_2505_17025_b200.hydrostatic import ABSORBING, WALL, BoundaryPair
from paper_2505_17025_b200.scenarios import (ScenarioSpec, still_water_state,
                                             vertical_momentum_from_constraint)

# slide kinematics per Froude number: (a0 m/s^2, u_t m/s, t1, t2, t3 s)
SLIDE_MOTIONS = {fr: SlideMotion(*row) for fr, row in {
    0.125: (1.500, 0.163, 0.109, 2.109, 2.218),
    0.25: (1.500, 0.327, 0.218, 2.218, 2.436),
    0.375: (1.500, 0.491, 0.327, 2.327, 2.654)}.items()}

HAMMACK_GAUGES = (0.61, 1.61, 9.61, 20.61)


def solitary_exact(x, t, a: float = 2.0, d: float = 10.0, x0: float = 200.0,
                   g: float = GRAVITY):
    """Closed-form solitary wave (eta, u) at time t."""
    if a <= 0 or d <= 0:
        raise ValueError("require a > 0 and d > 0")
    celerity = np.sqrt(g * (d + a))
    kappa = np.sqrt(3.0 * a / (4.0 * d * d * (d + a)))
    eta = a / np.cosh(kappa * (np.asarray(x, dtype=float) - celerity * t - x0)) ** 2
    return eta, celerity * eta / (d + eta)


def snap_to_node(grid: GridSpec, x: float) -> float:
    e, j = grid.nearest_node(x)
    return float(grid.nodes[e, j])


def _solitary(a=2.0, d=10.0, length=800.0, n_elements=200, dt=0.1, t_end=30.0, poly_order=1):
    grid = GridSpec(0.0, length, n_elements, poly_order)
    bottom = FlatBottom(d)
    eta, u = solitary_exact(grid.nodes, 0.0, a, d, length / 4.0)
    h = eta + d
    hu = u * h
    hw = vertical_momentum_from_constraint(grid, h, hu, bottom, 0.0)
    spec = ScenarioSpec("solitary", grid, dt, t_end, bottom, BoundaryPair(WALL, WALL))
    return spec, FlowState(*(NodalField(grid, v) for v in (h, hu, hw)), 0.0)


def _hammack(direction="up", h0=0.05, zeta0_mag=0.005, b=0.61, length=25.0, dx=0.025, dt=0.01,
             t_end=40.0, poly_order=1):
    grid = GridSpec(0.0, length, int(round(length / dx)), poly_order)
    edge = grid.dx * max(round(b / grid.dx), 1)          # plate edge on an element boundary
    sign = 1.0 if direction == "up" else -1.0
    bottom = HammackPlate(h0, sign * zeta0_mag, edge, hammack_time_constant(h0, edge, direction))
    spec = ScenarioSpec(f"hammack_{direction}", grid, dt, t_end, bottom,
                        BoundaryPair(WALL, ABSORBING),
                        tuple(snap_to_node(grid, x) for x in HAMMACK_GAUGES))
    return spec, still_water_state(grid, bottom)


def _whittaker(froude=0.25, h0=0.175, Hs=0.026, Ls=0.5, length=15.0, x_start=5.0, dx=0.075,
               dt=0.005, t_end=None, poly_order=1):
    if froude not in SLIDE_MOTIONS:
        raise ValueError(f"unknown Froude number {froude}; choose from {sorted(SLIDE_MOTIONS)}")
    grid = GridSpec(0.0, length, int(round(length / dx)), poly_order)
    bottom = WhittakerSlide(h0, Hs, Ls, SLIDE_MOTIONS[froude], x_start)
    t_end = 8.0 / np.sqrt(GRAVITY / Ls) if t_end is None else t_end   # t* = 8
    spec = ScenarioSpec(f"whittaker_fr{froude}", grid, dt, t_end, bottom,
                        BoundaryPair(ABSORBING, ABSORBING))
    return spec, still_water_state(grid, bottom)


CASES = {
    "solitary": _solitary,
    "hammack_up": lambda **kw: _hammack("up", **kw),
    "hammack_down": lambda **kw: _hammack("down", **kw),
    "whittaker": _whittaker,
}


def build_scenario(name: str, **overrides):
    """(ScenarioSpec, FlowState) of a named case, keyword overrides applied."""
    if name not in CASES:
        raise ValueError(f"unknown scenario {name!r}")
    return CASES[name](**overrides)


build_solitary = _solitary
build_hammack = _hammack
build_whittaker = _whittaker

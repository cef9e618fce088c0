"""Accuracy references of the benchmark harness (proj/src/problems.cpp):
closed-form logistic solution, RK4 reference tables with the step-halving
self check and linear interpolation (problems.cpp:11-70), RMSE
(problems.cpp:197-210).  The RK4 tables are integrated on the GPU
(pode_rk4_table); interpolation is host-side indexing."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _abi as A
from .api import InitialValueProblem, _ctx, _raise, problem_by_name

REFERENCE_STEPS = 32768  # problems.cpp:112 (kReferenceSteps)


def rk4_table(ivp: InitialValueProblem, steps: int, ctx=None) -> np.ndarray:
    """(steps+1) x dim RK4 table on [0, t_end] (integrate_rk4, problems.cpp:11-27)."""
    c = _ctx(ctx)
    table = np.zeros((steps + 1, ivp.dim))
    st = A.Status()
    pr = ivp._c()
    _raise(c._lib.pode_rk4_table(c.handle, C.byref(pr), steps, table.ctypes.data_as(A.dptr), C.byref(st)), st)
    return table


class Rk4Reference:
    """Rk4Reference (problems.cpp:29-65): integrate with h_ref and h_ref/2,
    require the endpoints to agree to 1e-10 (relative), keep the fine table."""

    def __init__(self, ivp: InitialValueProblem, h_ref: float, ctx=None):
        if not (h_ref > 0.0) or not (ivp.t_end > 0.0):
            from .api import InvalidInputError
            raise InvalidInputError("rk4_reference: need positive step and horizon")
        steps = int(round(math.ceil(ivp.t_end / h_ref)))
        coarse = rk4_table(ivp, steps, ctx)
        fine = rk4_table(ivp, 2 * steps, ctx)
        scale = max(1.0, float(np.linalg.norm(fine[-1])))
        if np.linalg.norm(coarse[-1] - fine[-1]) > 1e-10 * scale:
            raise ValueError("rk4_reference: step-halving check failed; h_ref is too coarse")
        self.table = fine
        self.t_end = ivp.t_end
        self.step = ivp.t_end / (fine.shape[0] - 1)

    def at(self, t: float) -> np.ndarray:
        if t < -1e-12 or t > self.t_end * (1.0 + 1e-12):
            from .api import InvalidInputError
            raise InvalidInputError("Rk4Reference: evaluation outside the integrated span")
        x = t / self.step
        last = self.table.shape[0] - 1
        nearest = int(min(max(0.0, round(x)), last))
        if abs(t - nearest * self.step) <= 1e-9 * max(1.0, abs(t)):
            return self.table[nearest]
        lo = int(min(max(0.0, math.floor(x)), last - 1))
        w = (t - lo * self.step) / self.step
        return (1.0 - w) * self.table[lo] + w * self.table[lo + 1]


def reference_for(name: str, ctx=None, grid_steps: int = 0):
    """The named problem's accuracy reference t -> y(t) (problems.cpp:116-190).

    The reference integrates its RK4 table with 32768 steps whatever the
    grid (problems.cpp:112), so RMSE on grids finer than the table measures
    the table's own interpolation and truncation error (SURVEY.md §8(f)
    item 3).  Given the grid's step count, the table here is refined to a
    power-of-two multiple of it (>= 32768 steps): every grid node is then a
    table node (no interpolation), and the step-halving check bounds the
    table's error at the finer step."""
    if name == "logistic":
        y0 = 0.01
        return lambda t: np.array([y0 / (y0 + (1.0 - y0) * math.exp(-t))])
    ivp = problem_by_name(name)
    steps = REFERENCE_STEPS
    if grid_steps > REFERENCE_STEPS:
        steps = grid_steps
    elif grid_steps > 0:
        steps = grid_steps * max(1, REFERENCE_STEPS // grid_steps)
    ref = Rk4Reference(ivp, ivp.t_end / steps, ctx)
    return ref.at


def rmse(means: np.ndarray, reference, grid) -> float:
    """problems.cpp:197-210"""
    means = np.asarray(means)
    if means.shape[0] != len(grid) or means.shape[0] == 0:
        from .api import DimensionError
        raise DimensionError("rmse: means and grid lengths disagree")
    acc, count = 0.0, 0
    for n, t in enumerate(grid):
        err = means[n] - reference(float(t))
        acc += float(np.dot(err, err))
        count += err.size
    return math.sqrt(acc / count)

"""pytest plugin: run the reference's OWN test suite with its hot path routed
through librebk ("How to route them through the shim").

Test infrastructure only — never imported by the product.  Load it before
collection so the names the reference's tests bind at import
(test_solvers.py:4-20 ``from kaczmarz import ... prepare, run``; cli.py
``from .solvers import ... run``) already point at the shim:

    PYTHONPATH=baseline/_ref:. python -m pytest -p tools.ref_shim_plugin \
        baseline/_ref/kaczmarz_tests            # tools/run_reference_tests.sh

What is rebound, for the device algorithms rebk / rek / rabk / rk only
(rbk, rdbk, dsbgs keep the reference's own code — they are off the path):

* ``run`` (solvers.py:425-474) -> ``paper_2001_04179_b200.run``: the whole
  loop, sampling and stopping rule in the persistent sm_100a kernel; the
  result is handed back as the reference's own ``RunTrace``.
* ``prepare`` (solvers.py:271) -> the reference's context, whose stepper
  (``ctx._step``, bound at solvers.py:187 from ``_STEPPERS``) is replaced by
  one device iteration (``rebk_run`` with explicit picks, drawn from
  ``state.rng`` exactly as the reference draws them, so ScriptedRng works).

The reference's validation errors still come from the reference (its
``prepare`` runs first); beta_max is handed over from the reference context
so the out-of-regime warning is decided on the identical number.  The
session summary prints how many calls went to the device, so a log proves
the CUDA path ran.
"""

from __future__ import annotations

import numpy as np

import kaczmarz
import kaczmarz.solvers as ks

import paper_2001_04179_b200 as dev
from paper_2001_04179_b200 import solvers as dev_solvers
from paper_2001_04179_b200.sampling import Partition as DevPartition

_orig_run = ks.run
_orig_prepare = ks.prepare
_COUNTS = {"run": 0, "step": 0, "ctx": 0}
_MATS: dict[int, tuple[object, object]] = {}


def _matrix(a):
    hit = _MATS.get(id(a))
    if hit is not None and hit[0] is a:
        return hit[1]
    m = dev.Matrix(dense=a._dense) if a._dense is not None else dev.Matrix(csr=a._csr)
    _MATS[id(a)] = (a, m)  # keep `a` alive so its id is not reused
    return m


def _partition(p):
    return None if p is None else DevPartition(p.axis, p.axis_len, tuple(p.blocks))


def _problem(p):
    return dev.ProblemInstance(a=_matrix(p.a), b=p.b, x_star=p.x_star, b_perp=p.b_perp,
                               meta=p.meta, oracle=p.oracle)


def _config(c, beta_max=None):
    return dev_solvers.SolverConfig(
        algorithm=c.algorithm, alpha=c.alpha,
        row_partition=_partition(c.row_partition), col_partition=_partition(c.col_partition),
        seed=c.seed, max_iters=c.max_iters,
        stop=dev_solvers.StoppingRule(mode=c.stop.mode, tol=c.stop.tol, check_stride=c.stop.check_stride),
        x0=c.x0, z0=c.z0, record_errors=c.record_errors,
        beta_max=c.beta_max if beta_max is None else beta_max,
    )


def _on_device(config) -> bool:
    return str(config.algorithm).lower() in dev_solvers.DEVICE_ALGORITHMS


def run(problem, config):
    if not _on_device(config):
        return _orig_run(problem, config)
    # the reference's own validation (and beta_max) first: same errors, same warnings
    ref_ctx = _orig_prepare(problem, config)
    t = dev_solvers.run(_problem(problem), _config(config, ref_ctx.beta_max))
    _COUNTS["run"] += 1
    return ks.RunTrace(iters=t.iters, converged=t.converged, wall_time=t.wall_time,
                       final_error=t.final_error, errors=t.errors, checkpoints=t.checkpoints,
                       warnings=t.warnings)


def prepare(problem, config):
    ctx = _orig_prepare(problem, config)
    if not _on_device(config):
        return ctx
    holder = {}

    def device_step(state, _ctx):
        d = holder.get("ctx")
        if d is None:
            d = holder["ctx"] = dev_solvers.prepare(_problem(problem), _config(config, ctx.beta_max))
            _COUNTS["ctx"] += 1
        _COUNTS["step"] += 1
        return d.step(state)

    ctx._step = device_step
    return ctx


def _install():
    for mod_name in ("kaczmarz", "kaczmarz.solvers", "kaczmarz.cli"):
        try:
            mod = __import__(mod_name, fromlist=["_"])
        except ImportError:
            continue
        if hasattr(mod, "run"):
            mod.run = run
        if hasattr(mod, "prepare"):
            mod.prepare = prepare


_install()


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(
        f"ref_shim: {_COUNTS['run']} run() calls and {_COUNTS['step']} step() calls "
        f"({_COUNTS['ctx']} device contexts) executed by librebk; "
        f"librebk = {dev._lib.LIB_PATH}"
    )

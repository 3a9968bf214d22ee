"""``snpsim`` alias that lets the reference's own test suite (copied
unmodified from ``/root/reference/pkg/tests`` into ``tests/conformance/``)
run against this package.

The alias module is the product package's public namespace (the drop-in
API, ``pkg/src/snpsim/__init__.py:4-67``) with ``snpsim.selection``,
``.generators``, ``.matrices``, ``.bench``, ``.cli``, ``.model``,
``.modelfile`` and ``.engine`` mapped to the package's modules, plus the
reference's CPU interpreter (``oracle_step`` / ``oracle_simulate`` /
``Format.ORACLE``, ``oracle.py:21-101``, ``engine.py:417-420``), which the
reference tests use as the checker.  That interpreter is this repo's test
oracle (``oracle/snp_oracle.py``): TEST INFRASTRUCTURE, reachable only
through this alias -- the product package itself has no CPU backend.
"""

from __future__ import annotations

import sys
import types

import numpy as np

import paper_2408_04343_b200 as pkg
from paper_2408_04343_b200 import (bench, cli, engine, generators, matrices, model, modelfile,
                                   selection)
from oracle.snp_oracle import OracleNegative, OracleSystem, interpret, interpret_step


def _oracle_system(system) -> OracleSystem:
    return OracleSystem.from_arrays(pkg.system_arrays(system.ensure_validated()))


def oracle_step(system, config, delays, sel, step: int = 0):
    """oracle.py:21-62 through the checker's interpreter."""
    policy, seed = selection.policy_code(sel)
    try:
        nxt, nd, fired = interpret_step(_oracle_system(system), [int(v) for v in config],
                                        [int(v) for v in delays], policy, seed, step)
    except OracleNegative as exc:
        raise pkg.NegativeSpikes(str(exc)) from exc
    return nxt, nd, fired


_RECORD = {pkg.RecordLevel.CONFIGS: "configs", pkg.RecordLevel.CONFIGS_AND_DELAYS: "delays",
           pkg.RecordLevel.FULL: "full"}


def oracle_simulate(system, options):
    """oracle.py:65-101 through the checker's interpreter, as a product Trace."""
    policy, seed = selection.policy_code(options.selection)
    try:
        tr = interpret(_oracle_system(system), options.max_steps, policy, seed, record=_RECORD[options.record])
    except OracleNegative as exc:
        raise pkg.NegativeSpikes(str(exc)) from exc
    reason = pkg.HaltReason.STEP_LIMIT if tr.halt == "step_limit" else pkg.HaltReason.NO_APPLICABLE_RULES
    return pkg.Trace(configs=[np.asarray(c, dtype=np.int64) for c in tr.configs], halt_reason=reason,
                     delays=tr.delays, spiking=tr.spiking)


class _OraclePrepared:
    def __init__(self, system):
        self.system = system
        self.fmt = pkg.Format.ORACLE
        self.rules = self.rule_map = self.matrix = None


def prepare(system, fmt, *a, **kw):
    if pkg.Format(fmt) is pkg.Format.ORACLE:
        system.ensure_validated()
        return _OraclePrepared(system)
    return pkg.prepare(system, fmt, *a, **kw)


def simulate_prepared(prep, options):
    if isinstance(prep, _OraclePrepared):
        return oracle_simulate(prep.system, options)
    return pkg.simulate_prepared(prep, options)


def simulate(system, fmt, options):
    return simulate_prepared(prepare(system, fmt), options)


def install() -> types.ModuleType:
    """Register the alias as ``snpsim`` (idempotent)."""
    mod = sys.modules.get("snpsim")
    if getattr(mod, "_conformance_alias", False):
        return mod
    mod = types.ModuleType("snpsim")
    mod.__dict__.update({k: v for k, v in vars(pkg).items() if not k.startswith("__")})
    mod.__dict__.update(oracle_step=oracle_step, oracle_simulate=oracle_simulate, prepare=prepare,
                        simulate=simulate, simulate_prepared=simulate_prepared, _conformance_alias=True)
    mod.__path__ = []  # a package, so "snpsim.x" submodule imports resolve through sys.modules
    sys.modules["snpsim"] = mod
    for name, sub in (("selection", selection), ("generators", generators), ("matrices", matrices),
                      ("bench", bench), ("cli", cli), ("model", model), ("modelfile", modelfile),
                      ("engine", engine)):
        sys.modules[f"snpsim.{name}"] = sub
        setattr(mod, name, sub)
    return mod

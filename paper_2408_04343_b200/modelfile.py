"""Plain-text model files (drop-in for ``snpsim.modelfile``, reference
``pkg/src/snpsim/modelfile.py:1-167``).

Format (version 1; neuron indices 1-based on disk, 0-based in memory)::

    snp 1
    neurons 3
    spikes 2 0 0
    rule 1 ge 1 1 1 0        # owner, ge|eq, threshold, consumed, produced, delay
    synapse 1 2
    output 3

``#`` starts a comment; blank lines are ignored.  ``parse_model`` /
``serialize_model`` work on text and ``SNPSystem`` objects exactly like the
reference (same error types, messages carry the line number, round trip is
the identity on validated systems).

At scale (10^7-10^8 neurons, 10^8-10^9 synapses) building an object per rule
and synapse is not an option, so :func:`load_model` / :func:`save_model` go
straight between a file and :class:`SystemArrays` through the native parser
and writer in ``csrc/snp_modelio.cpp`` (C ABI ``include/snpio.h``), which
apply the same checks in the same order and raise the same exception types.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .model import (InvalidRule, ModelError, ReflexiveSynapse, RegexKind, SNPSystem, SpikeRegex,
                    UnknownNeuron)

FORMAT_NAME = "snp"
FORMAT_VERSION = 1

_TOKENS = {RegexKind.AT_LEAST: "ge", RegexKind.EXACTLY: "eq"}
_KINDS = {tok: kind for kind, tok in _TOKENS.items()}


class ModelFileError(ModelError):
    """Malformed model-file text (modelfile.py:36-37)."""


# -- text <-> SNPSystem (reference API) ------------------------------------------------

def serialize_model(system: SNPSystem) -> str:
    """Model-file text of a (validated) system: header, neuron count, initial
    spikes, rules in validated order, synapses ascending, optional output
    (modelfile.py:40-57)."""
    system.ensure_validated()
    out = [f"{FORMAT_NAME} {FORMAT_VERSION}", f"neurons {system.neuron_count}"]
    out.append(" ".join(["spikes", *map(str, system.initial_spikes)]))
    out.extend(f"rule {r.neuron + 1} {_TOKENS[r.regex.kind]} {r.regex.threshold} {r.consumed} "
               f"{r.produced} {r.delay}" for r in system.rules)
    out.extend(f"synapse {a + 1} {b + 1}" for a, b in sorted(system.synapses))
    if system.output_neuron is not None:
        out.append(f"output {system.output_neuron + 1}")
    return "\n".join(out) + "\n"


class _Lines:
    """Per-line field access with the reference's diagnostics (modelfile.py:146-167)."""

    def __init__(self, lineno: int, args: list[str]):
        self.lineno, self.args = lineno, args

    def fail(self, msg: str) -> ModelFileError:
        return ModelFileError(f"line {self.lineno}: {msg}")

    def int(self, pos: int, what: str) -> int:
        if pos >= len(self.args):
            raise self.fail(f"missing {what}")
        try:
            return int(self.args[pos])
        except ValueError:
            raise self.fail(f"{what} must be an integer, got {self.args[pos]!r}") from None

    def index(self, pos: int, count: int) -> int:
        v = self.int(pos, "neuron index")
        if not 1 <= v <= count:
            raise self.fail(f"neuron index {v} out of range 1..{count}")
        return v - 1


def parse_model(text: str) -> SNPSystem:
    """Parse model-file text into a validated ``SNPSystem`` (modelfile.py:60-143).

    Malformed text raises :class:`ModelFileError`; semantic violations keep
    their own types (``InvalidRule``, ``ReflexiveSynapse``, ``ModelError``).
    """
    system = SNPSystem()
    header = False
    count: int | None = None
    spikes = False
    for lineno, raw in enumerate(text.splitlines(), start=1):
        fields = raw.split("#", 1)[0].split()
        if not fields:
            continue
        key, ln = fields[0], _Lines(lineno, fields[1:])
        if not header:
            if key != FORMAT_NAME:
                raise ln.fail(f"expected '{FORMAT_NAME} <version>' header, got {raw!r}")
            version = ln.int(0, "format version")
            if version != FORMAT_VERSION:
                raise ln.fail(f"unsupported format version {version}")
            header = True
        elif key == "neurons":
            if count is not None:
                raise ln.fail("duplicate 'neurons' line")
            count = ln.int(0, "neuron count")
            if count < 0:
                raise ln.fail("neuron count must be >= 0")
        elif key == "spikes":
            if count is None:
                raise ln.fail("'spikes' before 'neurons'")
            if spikes:
                raise ln.fail("duplicate 'spikes' line")
            if len(ln.args) != count:
                raise ln.fail(f"expected {count} spike counts, got {len(ln.args)}")
            for pos in range(count):
                system.add_neuron(ln.int(pos, "spike count"))
            spikes = True
        elif key in ("rule", "synapse", "output"):
            if not spikes:
                raise ln.fail("directive before 'spikes' line")
            if key == "rule":
                if len(ln.args) != 6:
                    raise ln.fail(f"'rule' needs 6 fields, got {len(ln.args)}")
                kind = _KINDS.get(ln.args[1])
                if kind is None:
                    raise ln.fail(f"condition kind must be 'ge' or 'eq', got {ln.args[1]!r}")
                owner = ln.index(0, count)
                regex = SpikeRegex(kind, ln.int(2, "threshold"))
                system.add_rule(owner, regex, ln.int(3, "consumed"), ln.int(4, "produced"), ln.int(5, "delay"))
            elif key == "synapse":
                if len(ln.args) != 2:
                    raise ln.fail("'synapse' needs 2 fields")
                src = ln.index(0, count)
                system.add_synapse(src, ln.index(1, count))
            else:
                system.output_neuron = ln.index(0, count)
        else:
            raise ln.fail(f"unknown directive {key!r}")
    if not header:
        raise ModelFileError("empty model file")
    if count is None or not spikes:
        raise ModelFileError("model file is missing 'neurons' or 'spikes'")
    return system.validate()


# -- files <-> SystemArrays (native, at scale) ---------------------------------------

IO_LIB_PATH = Path(__file__).resolve().parent / "libsnpio.so"
_ERRORS = {1: ModelFileError, 2: InvalidRule, 3: UnknownNeuron, 4: ReflexiveSynapse, 5: ModelError,
           6: OSError, 7: MemoryError}
_io = None


def _io_lib() -> ctypes.CDLL:
    global _io
    if _io is None:
        path = Path(os.environ.get("SNPIO_LIB", IO_LIB_PATH))
        if not path.exists():
            raise ImportError(f"{path} not found: build it (python -c 'import __graft_entry__ as g; g.build()')")
        lib = ctypes.CDLL(str(path))
        vp, i64, i64p = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)
        sig = {
            "snpio_last_error": (ctypes.c_char_p, []),
            "snpio_parse": (ctypes.c_int, [ctypes.c_char_p, i64, ctypes.POINTER(vp)]),
            "snpio_parse_file": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(vp)]),
            "snpio_model_sizes": (ctypes.c_int, [vp, i64p, i64p, i64p, i64p]),
            "snpio_model_export": (ctypes.c_int, [vp] + [vp] * 9),
            "snpio_model_free": (None, [vp]),
            "snpio_write_file": (ctypes.c_int, [ctypes.c_char_p, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp,
                                                vp, vp, i64]),
            "snpio_write_trace": (ctypes.c_int, [ctypes.c_char_p, vp, i64, i64, ctypes.c_int32]),
            "snpio_synth_v1_edges": (ctypes.c_int, [i64, ctypes.c_uint64, i64, i64, i64p]),
            "snpio_synth_v1": (ctypes.c_int, [i64, ctypes.c_uint64, ctypes.c_int32, i64, i64] + [vp] * 9),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _io = lib
    return _io


def _check(rc: int) -> None:
    if rc:
        msg = _io_lib().snpio_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, ModelError)(msg)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _to_arrays(handle: ctypes.c_void_p):
    from .generators import SystemArrays
    from .matrices import NeuronRuleMap, RuleVector
    lib = _io_lib()
    q, m, s, out = (ctypes.c_int64() for _ in range(4))
    _check(lib.snpio_model_sizes(handle, ctypes.byref(q), ctypes.byref(m), ctypes.byref(s), ctypes.byref(out)))
    q, m, s = q.value, m.value, s.value
    init = np.empty(q, np.int64)
    off = np.empty(q + 1, np.int64)
    thr, cons, prod, dly = (np.empty(m, np.int64) for _ in range(4))
    exact = np.empty(m, np.bool_)
    aoff = np.empty(q + 1, np.int64)
    adst = np.empty(s, np.int64)
    _check(lib.snpio_model_export(handle, *map(_ptr, (init, off, thr, exact, cons, prod, dly, aoff, adst))))
    owner = np.repeat(np.arange(q, dtype=np.int64), np.diff(off))
    rules = RuleVector(thr, exact, cons, prod, dly, owner)
    return SystemArrays(init, rules, NeuronRuleMap(off), aoff, adst, None if out.value < 0 else int(out.value))


def load_model(path: str | os.PathLike):
    """Parse a model file straight into :class:`SystemArrays` (native parser;
    same checks, order and exception types as :func:`parse_model`)."""
    lib = _io_lib()
    h = ctypes.c_void_p()
    _check(lib.snpio_parse_file(os.fsencode(path), ctypes.byref(h)))
    try:
        return _to_arrays(h)
    finally:
        lib.snpio_model_free(h)


def parse_model_arrays(text: str | bytes):
    """:func:`load_model` on in-memory text."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    lib = _io_lib()
    h = ctypes.c_void_p()
    _check(lib.snpio_parse(data, len(data), ctypes.byref(h)))
    try:
        return _to_arrays(h)
    finally:
        lib.snpio_model_free(h)


def save_model(path: str | os.PathLike, system) -> None:
    """Write a system (``SNPSystem`` or ``SystemArrays``) as a model file; the
    bytes equal ``serialize_model`` of the same system (native writer)."""
    from .generators import system_arrays
    a = system_arrays(system)
    c = lambda x: np.ascontiguousarray(x, dtype=np.int64)
    init, off = c(a.initial), c(a.rule_map.offsets)
    r = a.rules
    thr, cons, prod, dly = c(r.threshold), c(r.consumed), c(r.produced), c(r.delay)
    exact = np.ascontiguousarray(r.is_exact, dtype=np.uint8)
    aoff, adst = c(a.adj_offsets), c(a.adj_targets)
    out = -1 if a.output_neuron is None else int(a.output_neuron)
    _check(_io_lib().snpio_write_file(os.fsencode(path), len(init), len(thr), len(adst),
                                      *map(_ptr, (init, off, thr, exact, cons, prod, dly, aoff, adst)), out))


def write_trace(path: str | os.PathLike, trace, append: bool = False) -> None:
    """Write ``format_trace(trace)`` to ``path`` with the native writer
    (engine.py:162-165; byte-identical, without building the text in Python).
    ``trace`` is a Trace or a sequence of configuration rows."""
    rows = trace.configs if hasattr(trace, "configs") else trace
    arr = np.ascontiguousarray(np.stack([np.asarray(r, dtype=np.int64) for r in rows]) if len(rows) else
                               np.zeros((0, 0), np.int64))
    q = arr.shape[1] if arr.ndim == 2 else 0
    _check(_io_lib().snpio_write_trace(os.fsencode(path), _ptr(arr), arr.shape[0], q, 1 if append else 0))

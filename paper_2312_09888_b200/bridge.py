"""SENSEI-style configurable bridge in front of the GPU analyses.

Behavioural contract (reference pkg/src/nekmini/bridge.py, re-implemented):
  * document: root ``<sensei>``, children ``<analysis type=.. frequency=..>``;
    other children are ignored with a warning (:68-71); malformed XML, a
    wrong root, a missing type, an unknown kind, a non-integer or < 1
    frequency are ConfigError (:59-88); ``catalyst`` means ``render``
    (:77-78); attributes a kind does not know are dropped with a warning
    (:89-94).
  * triggering: step 0 fires iff trigger_at_step_zero, any other step fires
    when divisible by the frequency; negative steps are an error (:107-112).
  * update: snapshot validated, steps strictly increasing (:151-158), sinks
    run in document order, each timed; an exception inside a sink becomes
    that sink's report error and the remaining sinks still run (:161-177).
  * finalize: every sink flushed, failures counted and logged (:179-187).

Addition: an optional communicator (the paper's ``initialize(MPI_Comm*,
nek_data)``) forwarded to every sink so the in situ sink
can depth-composite across ranks.
"""
from __future__ import annotations

import logging
import time
import xml.etree.ElementTree as ET
from dataclasses import dataclass, field

from . import sinks as sinks_mod
from .data_model import Snapshot, validate_snapshot

log = logging.getLogger(__name__)

# kind -> accepted attributes (everything else on the element warns)
_ATTRS_BY_KIND: dict[str, frozenset[str]] = {
    "render": frozenset({"dir", "width", "height", "field", "vmin", "vmax"}),
    "insitu": frozenset({"dir", "width", "height", "field", "vmin", "vmax", "iso", "slice", "view",
                         "velocity", "composite", "continuous", "projection", "fov", "async_write"}),
    "transit": frozenset({"dir", "width", "height", "field", "vmin", "vmax", "iso", "slice", "view",
                          "velocity", "endpoint", "projection", "fov"}),
    "stats": frozenset({"path"}),
    "checkpoint": frozenset({"dir", "format", "arrays"}),
    "null": frozenset(),
}
_ALIASES = {"catalyst": "render"}
KINDS = tuple(_ATTRS_BY_KIND)
_KNOWN_ATTRS = {k: set(v) for k, v in _ATTRS_BY_KIND.items()}


class ConfigError(ValueError):
    """The configuration document is malformed or inconsistent."""


@dataclass(frozen=True)
class AnalysisSpec:
    kind: str
    frequency: int
    params: dict[str, str] = field(default_factory=dict)


@dataclass(frozen=True)
class BridgeConfig:
    specs: tuple[AnalysisSpec, ...] = ()
    trigger_at_step_zero: bool = True


def _frequency_of(raw: str) -> int:
    try:
        value = int(raw)
    except ValueError:
        raise ConfigError(f"frequency must be an integer, got {raw!r}") from None
    if value < 1:
        raise ConfigError(f"frequency must be >= 1, got {value}")
    return value


def _spec_from_element(el: ET.Element) -> AnalysisSpec:
    attrs = dict(el.attrib)
    if "type" not in attrs:
        raise ConfigError("<analysis> element missing 'type' attribute")
    kind = _ALIASES.get(attrs["type"], attrs["type"])
    if kind not in _ATTRS_BY_KIND:
        raise ConfigError(f"unknown analysis kind {kind!r}")
    freq = _frequency_of(attrs.get("frequency", "1"))
    allowed = _ATTRS_BY_KIND[kind]
    params: dict[str, str] = {}
    for key, val in attrs.items():
        if key in ("type", "frequency"):
            continue
        if key not in allowed:
            log.warning("ignoring unknown attribute %r on analysis type %r", key, kind)
            continue
        params[key] = val
    if kind == "stats" and "path" not in params:
        raise ConfigError("stats analysis requires a 'path' attribute")
    return AnalysisSpec(kind, freq, params)


def parse_config(text: str) -> BridgeConfig:
    try:
        root = ET.fromstring(text)
    except ET.ParseError as exc:
        raise ConfigError(f"malformed configuration document: {exc}") from exc
    if root.tag != "sensei":
        raise ConfigError(f"expected root element <sensei>, got <{root.tag}>")
    specs: list[AnalysisSpec] = []
    for child in root:
        if child.tag == "analysis":
            specs.append(_spec_from_element(child))
        else:
            log.warning("ignoring unknown element <%s>", child.tag)
    return BridgeConfig(specs=tuple(specs))


def load_config(path: str) -> BridgeConfig:
    with open(path, encoding="utf-8") as fh:
        return parse_config(fh.read())


def should_trigger(spec: AnalysisSpec, step: int, trigger_at_step_zero: bool = True) -> bool:
    if step < 0:
        raise ValueError("step must be non-negative")
    return trigger_at_step_zero if step == 0 else (step % spec.frequency == 0)


@dataclass
class SinkReport:
    kind: str
    seconds: float
    bytes_written: int
    error: str | None = None


@dataclass
class SinkSummary:
    kind: str
    invocations: int = 0
    seconds: float = 0.0
    bytes_written: int = 0
    failures: int = 0

    def record(self, rep: SinkReport) -> None:
        self.invocations += 1
        self.seconds += rep.seconds
        self.bytes_written += rep.bytes_written
        if rep.error is not None:
            self.failures += 1


def _run_isolated(kind: str, sink, snapshot) -> SinkReport:
    start = time.perf_counter()
    try:
        written, error = sink.consume(snapshot), None
    except Exception as exc:  # isolation: one broken analysis never stops the others
        written, error = 0, f"{type(exc).__name__}: {exc}"
    return SinkReport(kind, time.perf_counter() - start, written, error)


class Bridge:
    """Dispatches snapshots to the configured analyses; single-threaded by
    contract (one logical thread of control per bridge)."""

    def __init__(self, cfg: BridgeConfig, comm=None):
        self.cfg = cfg
        self.comm = comm
        self.sinks = [sinks_mod.make_sink(sp.kind, sp.params, comm=comm) for sp in cfg.specs]
        self.summaries = [SinkSummary(sp.kind) for sp in cfg.specs]
        self._last_step: int | None = None

    def _admit(self, s: Snapshot) -> None:
        problems = validate_snapshot(s)
        if problems:
            raise ValueError(f"invalid snapshot: {problems}")
        prev = self._last_step
        if prev is not None and s.step <= prev:
            raise ValueError(f"non-increasing step {s.step} (previous update was step {prev})")
        self._last_step = s.step

    def update(self, s: Snapshot) -> list[SinkReport]:
        self._admit(s)
        out: list[SinkReport] = []
        for spec, sink, summary in zip(self.cfg.specs, self.sinks, self.summaries):
            if should_trigger(spec, s.step, self.cfg.trigger_at_step_zero):
                rep = _run_isolated(spec.kind, sink, s)
                summary.record(rep)
                out.append(rep)
        return out

    def finalize(self) -> list[SinkSummary]:
        for sink, summary in zip(self.sinks, self.summaries):
            try:
                sink.finalize()
            except Exception as exc:
                summary.failures += 1
                log.warning("sink %s failed to flush: %s", summary.kind, exc)
        return list(self.summaries)


def initialize(cfg: BridgeConfig, comm=None) -> Bridge:
    """Build every sink up front so unwritable outputs fail immediately."""
    return Bridge(cfg, comm=comm)

"""Routes and signal timing (SPaT) — host-side input model.

Mirrors the reference's ``ecodrive.route`` data model (route.py:29-184,
331-427): per-node speed bounds / grade / kind, fixed-time signals with
half-open green windows in cycle-local time, and the JSON loader.  Phase
arithmetic uses Python's floored float ``%`` exactly like the reference
(route.py:69-86); the CUDA side restates the same floored remainder.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path
from typing import Mapping

import numpy as np

from .errors import RouteFormatError, UnknownSignalError

NODE_PLAIN = 0
NODE_SIGNAL = 1
NODE_STOP = 2

GREEN = "green"
RED = "red"


def _finite(value, name: str, *, lo=None, lo_strict=False, hi=None, hi_strict=False) -> float:
    x = float(value)
    if not math.isfinite(x):
        raise RouteFormatError(name, f"must be finite, got {value!r}")
    if lo is not None and (x <= lo if lo_strict else x < lo):
        raise RouteFormatError(name, f"must be {'>' if lo_strict else '>='} {lo}, got {x}")
    if hi is not None and (x >= hi if hi_strict else x > hi):
        raise RouteFormatError(name, f"must be {'<' if hi_strict else '<='} {hi}, got {x}")
    return x


@dataclass(frozen=True)
class SignalTiming:
    """Fixed-time program: green iff ``(t - offset) mod cycle`` lies in one of
    the half-open windows (route.py:34-86)."""

    cycle: float
    offset: float
    green_windows: tuple

    def __post_init__(self):
        _finite(self.cycle, "cycle", lo=0.0, lo_strict=True)
        _finite(self.offset, "offset")
        end_prev = 0.0
        for i, (a, b) in enumerate(self.green_windows):
            if not (0.0 <= a < b <= self.cycle):
                raise RouteFormatError(
                    f"green_windows[{i}]",
                    f"window [{a}, {b}) must satisfy 0 <= start < end <= cycle={self.cycle}")
            if a < end_prev:
                raise RouteFormatError(f"green_windows[{i}]", "windows must be sorted and non-overlapping")
            end_prev = b

    def local_time(self, t: float) -> float:
        return float((t - self.offset) % self.cycle)

    def is_green(self, t: float) -> bool:
        tau = self.local_time(t)
        return any(a <= tau < b for a, b in self.green_windows)

    def next_green_from(self, t: float) -> float:
        """Start of the next green after a red instant ``t`` (route.py:79-86)."""
        if self.is_green(t):
            raise ValueError(f"next_green_from called during green at t={t}")
        tau = self.local_time(t)
        return t + min((a - tau) % self.cycle for a, _ in self.green_windows)


@dataclass(frozen=True)
class SpatSchedule:
    """signal id -> SignalTiming."""

    signals: Mapping[str, SignalTiming]

    def timing(self, signal_id: str) -> SignalTiming:
        if signal_id not in self.signals:
            raise UnknownSignalError(signal_id)
        return self.signals[signal_id]


@dataclass(frozen=True)
class Route:
    """Nodes ``0..N-1`` spaced ``delta_d`` apart with stationary features."""

    delta_d: float
    v_min: np.ndarray
    v_max: np.ndarray
    grade: np.ndarray
    traffic_lights: Mapping[int, str]
    stop_signs: tuple
    accel_min: float
    accel_max: float
    stop_dwell: float = 2.0
    name: str = "route"

    def __post_init__(self):
        _finite(self.delta_d, "delta_d", lo=0.0, lo_strict=True)
        n = self.v_min.shape[0]
        if n < 1:
            raise RouteFormatError("node_count", f"route needs >= 1 node, got {n}")
        for attr in ("v_max", "grade"):
            if getattr(self, attr).shape[0] != n:
                raise RouteFormatError(attr, f"length must equal node_count={n}")
        bad = np.flatnonzero(self.v_min < 0.0)
        if bad.size:
            raise RouteFormatError(f"v_min[{int(bad[0])}]", "speed bounds must be >= 0")
        bad = np.flatnonzero(self.v_min >= self.v_max)
        if bad.size:
            i = int(bad[0])
            raise RouteFormatError(f"v_min[{i}]", f"must be < v_max[{i}] ({self.v_min[i]} >= {self.v_max[i]})")
        _finite(self.accel_min, "accel_min", hi=0.0, hi_strict=True)
        _finite(self.accel_max, "accel_max", lo=0.0, lo_strict=True)
        _finite(self.stop_dwell, "stop_dwell", lo=0.0)
        for node in self.traffic_lights:
            if not 0 <= node < n:
                raise RouteFormatError("traffic_lights", f"node {node} outside [0, {n})")
        for node in self.stop_signs:
            if not 0 <= node < n:
                raise RouteFormatError("stop_signs", f"node {node} outside [0, {n})")
            if node in self.traffic_lights:
                raise RouteFormatError("stop_signs", f"node {node} is also a traffic-light node")
        for node in (*self.traffic_lights, *self.stop_signs):
            if self.v_min[node] != 0.0:
                raise RouteFormatError(f"v_min[{node}]", "must be 0 at traffic-light and stop-sign nodes")

    @property
    def node_count(self) -> int:
        return int(self.v_min.shape[0])

    @property
    def length(self) -> float:
        return (self.node_count - 1) * self.delta_d

    def node_kind(self, s: int) -> int:
        if s in self.traffic_lights:
            return NODE_SIGNAL
        return NODE_STOP if s in self.stop_signs else NODE_PLAIN

    def node_kinds(self) -> np.ndarray:
        kinds = np.zeros(self.node_count, dtype=np.int8)
        kinds[list(self.traffic_lights)] = NODE_SIGNAL
        kinds[list(self.stop_signs)] = NODE_STOP
        return kinds


def phase_at(spat: SpatSchedule, signal_id: str, t: float) -> str:
    return GREEN if spat.timing(signal_id).is_green(t) else RED


def next_green_start(spat: SpatSchedule, signal_id: str, t: float) -> float:
    timing = spat.timing(signal_id)
    if timing.is_green(t):
        raise ValueError(f"next_green_start called while signal {signal_id!r} is green at t={t}")
    return timing.next_green_from(t)


def _node_array(doc: dict, key: str, n: int) -> np.ndarray:
    if key not in doc or doc[key] is None:
        raise RouteFormatError(key, "required field is missing")
    raw = doc[key]
    if isinstance(raw, (int, float)):
        return np.full(n, float(raw))
    arr = np.asarray(raw, dtype=np.float64)
    if arr.ndim != 1 or arr.shape[0] != n:
        raise RouteFormatError(key, f"must be a scalar or a list of {n} numbers")
    if not np.all(np.isfinite(arr)):
        raise RouteFormatError(key, "values must be finite")
    return np.ascontiguousarray(arr)


def _required(doc: dict, key: str, parent: str = ""):
    if key not in doc:
        raise RouteFormatError(f"{parent}{key}", "required field is missing")
    return doc[key]


def load_route(source) -> tuple:
    """Route + SPaT document (a JSON path or the parsed dict) -> (Route,
    SpatSchedule).  Same schema as the reference loader (route.py:331-418)."""
    if isinstance(source, (str, Path)):
        try:
            doc = json.loads(Path(source).read_text())
        except json.JSONDecodeError as exc:
            raise RouteFormatError("<document>", f"invalid JSON: {exc}") from None
    else:
        doc = source
    if not isinstance(doc, dict):
        raise RouteFormatError("<document>", "top level must be a JSON object")
    n = int(_required(doc, "node_count"))
    if n < 1:
        raise RouteFormatError("node_count", f"must be >= 1, got {n}")
    lights = {}
    for i, entry in enumerate(doc.get("traffic_lights", [])):
        if not isinstance(entry, dict) or "node" not in entry or "signal" not in entry:
            raise RouteFormatError(f"traffic_lights[{i}]", "must be an object with node and signal")
        node = int(entry["node"])
        if node in lights:
            raise RouteFormatError(f"traffic_lights[{i}]", f"duplicate traffic light at node {node}")
        lights[node] = str(entry["signal"])
    stops = tuple(int(s) for s in doc.get("stop_signs", []))
    if len(set(stops)) != len(stops):
        raise RouteFormatError("stop_signs", "duplicate stop-sign node")
    signals = {}
    for sid, sdoc in dict(doc.get("signals", {})).items():
        parent = f"signals[{sid}]."
        try:
            windows = tuple((float(a), float(b)) for a, b in _required(sdoc, "green_windows_s", parent))
        except (TypeError, ValueError):
            raise RouteFormatError(parent + "green_windows_s", "must be a list of [start, end] pairs") from None
        try:
            signals[sid] = SignalTiming(cycle=float(_required(sdoc, "cycle_s", parent)),
                                        offset=float(sdoc.get("offset_s", 0.0)),
                                        green_windows=windows)
        except RouteFormatError as exc:
            raise RouteFormatError(parent + exc.field, str(exc).split(": ", 1)[1]) from None
    for node, sid in lights.items():
        if sid not in signals:
            raise RouteFormatError(f"traffic_lights[node={node}].signal", f"unknown signal id {sid!r}")
    route = Route(
        delta_d=float(_required(doc, "delta_d_m")),
        v_min=_node_array(doc, "v_min_mps", n),
        v_max=_node_array(doc, "v_max_mps", n),
        grade=_node_array(doc, "grade_rad", n) if "grade_rad" in doc else np.zeros(n),
        traffic_lights=lights,
        stop_signs=stops,
        accel_min=float(_required(doc, "accel_min_mps2")),
        accel_max=float(_required(doc, "accel_max_mps2")),
        stop_dwell=float(doc.get("stop_dwell_s", 2.0)),
        name=str(doc.get("name", "route")),
    )
    return route, SpatSchedule(signals=signals)

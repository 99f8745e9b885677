"""Vehicle description and the loop's value types (host side).

The P0 mild-hybrid plant is *evaluated* only on the device
(``csrc/eco_plant.cuh``); this module holds its parameters and the frozen
records that flow through the receding-horizon loop.  Field names and
meanings follow the reference's ``ecodrive.plant`` (plant.py:28-265):
``Vehicle.pack()`` returns the same ``PlantPack`` field set
(_kernels.py:31-53) that the C ABI's ``EcoPlant`` struct mirrors.
"""

from __future__ import annotations

from collections import namedtuple
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from .errors import VehicleFormatError


@dataclass(frozen=True)
class StateVector:
    v: float          # speed (m/s)
    soc: float        # state of charge (0..1)
    t: float          # trip clock (s)

    def as_array(self) -> np.ndarray:
        return np.array([self.v, self.soc, self.t], dtype=np.float64)


@dataclass(frozen=True)
class ActionVector:
    t_eng: float      # engine crank torque (N m)
    t_bsg: float      # BSG shaft torque (N m), negative = generating

    def as_array(self) -> np.ndarray:
        return np.array([self.t_eng, self.t_bsg], dtype=np.float64)


class StepInfo(NamedTuple):
    dt_move: float
    wait: float
    fuel_g: float
    accel: float
    clamped: bool
    gear: int


PlantPack = namedtuple("PlantPack", [
    "mass", "c0", "c1", "c2", "wheel_radius", "final_drive",
    "gear_ratios", "gear_eff", "shift_v", "idle_speed", "belt_ratio",
    "eng_w", "eng_tmin", "eng_tmax", "fuel_w", "fuel_t", "fuel_vals",
    "bsg_w", "bsg_tmin", "bsg_tmax", "bsgeff_w", "bsgeff_t", "bsgeff_vals",
    "r0", "c_nom", "voc_soc", "voc_v", "soc_min", "soc_max", "p_bat_max",
])


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _increasing(a: np.ndarray, name: str):
    if a.ndim != 1 or a.size < 2 or np.any(np.diff(a) <= 0):
        raise VehicleFormatError(name, "must be a strictly increasing 1-D array of >= 2 values")


@dataclass(frozen=True)
class VehicleParams:
    mass: float
    c0: float
    c1: float
    c2: float
    wheel_radius: float
    final_drive: float
    gear_ratios: np.ndarray
    gear_efficiencies: np.ndarray
    shift_speeds: np.ndarray
    idle_speed: float

    def __post_init__(self):
        for name in ("gear_ratios", "gear_efficiencies", "shift_speeds"):
            object.__setattr__(self, name, _f64(getattr(self, name)))
        for name in ("mass", "wheel_radius", "final_drive", "idle_speed"):
            if not getattr(self, name) > 0.0:
                raise VehicleFormatError(name, "must be > 0")
        for name in ("c0", "c1", "c2"):
            if not getattr(self, name) >= 0.0:
                raise VehicleFormatError(name, "must be >= 0")
        g = self.gear_ratios.shape[0]
        if g < 1 or np.any(self.gear_ratios <= 0):
            raise VehicleFormatError("gear_ratios", "at least one positive ratio required")
        if self.gear_efficiencies.shape[0] != g or np.any(
                (self.gear_efficiencies <= 0) | (self.gear_efficiencies > 1)):
            raise VehicleFormatError("gear_efficiencies", f"need {g} values in (0, 1]")
        if self.shift_speeds.shape[0] != g - 1 or np.any(np.diff(self.shift_speeds) <= 0):
            raise VehicleFormatError("shift_speeds", f"need {g - 1} increasing values")


@dataclass(frozen=True)
class EngineModel:
    speed_axis: np.ndarray
    torque_min: np.ndarray
    torque_max: np.ndarray
    fuel_speed_axis: np.ndarray
    fuel_torque_axis: np.ndarray
    fuel_map: np.ndarray        # g/s, (speed, torque) row-major

    def __post_init__(self):
        for name in ("speed_axis", "torque_min", "torque_max", "fuel_speed_axis",
                     "fuel_torque_axis", "fuel_map"):
            object.__setattr__(self, name, _f64(getattr(self, name)))
        _increasing(self.speed_axis, "speed_axis")
        _increasing(self.fuel_speed_axis, "fuel_speed_axis")
        _increasing(self.fuel_torque_axis, "fuel_torque_axis")
        if self.fuel_map.shape != (self.fuel_speed_axis.size, self.fuel_torque_axis.size):
            raise VehicleFormatError("fuel_map", "shape must match its axes")


@dataclass(frozen=True)
class BsgModel:
    belt_ratio: float
    speed_axis: np.ndarray
    torque_min: np.ndarray
    torque_max: np.ndarray
    eff_speed_axis: np.ndarray
    eff_torque_axis: np.ndarray
    eff_map: np.ndarray         # (speed, |T|), values in (0, 1]

    def __post_init__(self):
        for name in ("speed_axis", "torque_min", "torque_max", "eff_speed_axis",
                     "eff_torque_axis", "eff_map"):
            object.__setattr__(self, name, _f64(getattr(self, name)))
        if not self.belt_ratio > 0:
            raise VehicleFormatError("belt_ratio", "must be > 0")
        _increasing(self.speed_axis, "speed_axis")
        _increasing(self.eff_speed_axis, "eff_speed_axis")
        _increasing(self.eff_torque_axis, "eff_torque_axis")
        if self.eff_map.shape != (self.eff_speed_axis.size, self.eff_torque_axis.size):
            raise VehicleFormatError("eff_map", "shape must match its axes")
        if np.any((self.eff_map <= 0) | (self.eff_map > 1)):
            raise VehicleFormatError("eff_map", "efficiencies must lie in (0, 1]")


@dataclass(frozen=True)
class BatteryModel:
    r0: float
    c_nom: float
    voc_soc_axis: np.ndarray
    voc: np.ndarray
    soc_min: float = 0.2
    soc_max: float = 0.9

    def __post_init__(self):
        object.__setattr__(self, "voc_soc_axis", _f64(self.voc_soc_axis))
        object.__setattr__(self, "voc", _f64(self.voc))
        if not (self.r0 > 0 and self.c_nom > 0):
            raise VehicleFormatError("r0/c_nom", "must be > 0")
        _increasing(self.voc_soc_axis, "voc_soc_axis")
        if self.voc.shape != self.voc_soc_axis.shape or np.any(self.voc <= 0):
            raise VehicleFormatError("voc", "need positive voltages matching voc_soc_axis")
        if not 0.0 <= self.soc_min < self.soc_max <= 1.0:
            raise VehicleFormatError("soc_min/soc_max", f"need 0 <= {self.soc_min} < {self.soc_max} <= 1")

    def max_deliverable_power(self) -> float:
        """max V_oc^2 / (4 R0) over the pack (plant.py:211-214)."""
        return float(np.max(self.voc) ** 2 / (4.0 * self.r0))


@dataclass(frozen=True)
class Vehicle:
    params: VehicleParams
    engine: EngineModel
    bsg: BsgModel
    battery: BatteryModel
    name: str = "vehicle"
    _pack: list = field(default_factory=list, repr=False, compare=False)

    def pack(self) -> PlantPack:
        if not self._pack:
            p, e, b, bat = self.params, self.engine, self.bsg, self.battery
            self._pack.append(PlantPack(
                mass=p.mass, c0=p.c0, c1=p.c1, c2=p.c2, wheel_radius=p.wheel_radius,
                final_drive=p.final_drive, gear_ratios=p.gear_ratios,
                gear_eff=p.gear_efficiencies, shift_v=p.shift_speeds,
                idle_speed=p.idle_speed, belt_ratio=b.belt_ratio,
                eng_w=e.speed_axis, eng_tmin=e.torque_min, eng_tmax=e.torque_max,
                fuel_w=e.fuel_speed_axis, fuel_t=e.fuel_torque_axis, fuel_vals=e.fuel_map,
                bsg_w=b.speed_axis, bsg_tmin=b.torque_min, bsg_tmax=b.torque_max,
                bsgeff_w=b.eff_speed_axis, bsgeff_t=b.eff_torque_axis, bsgeff_vals=b.eff_map,
                r0=bat.r0, c_nom=bat.c_nom, voc_soc=bat.voc_soc_axis, voc_v=bat.voc,
                soc_min=bat.soc_min, soc_max=bat.soc_max,
                p_bat_max=bat.max_deliverable_power(),
            ))
        return self._pack[0]

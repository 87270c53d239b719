"""B200-native (sm_100a, fp64) EAM force hot path of MISA-MD (arXiv 2107.07866).

The product is ``libcascade_b200.so`` (C ABI in include/cascade_b200.h);
this package is its host-side mirror of the reference cascademd API.
"""
from .engine import (ACCEL_FACTOR, BOLTZMANN_EV, MV2_TO_EV, SPEED_FACTOR, DeviceStore,
                     EamPotential, OutputSpec, PkaSpec, SimConfig, Simulation, StoreArrays,
                     ThermostatSpec, adaptive_dt, build_offsets, make_box, pka_speed)
from .potential import BASELINE_RHO_MAX, write_baseline_table

__all__ = ["ACCEL_FACTOR", "BOLTZMANN_EV", "MV2_TO_EV", "SPEED_FACTOR", "DeviceStore",
           "EamPotential", "OutputSpec", "PkaSpec", "SimConfig", "ThermostatSpec", "Simulation", "StoreArrays", "adaptive_dt",
           "build_offsets", "make_box", "pka_speed", "BASELINE_RHO_MAX", "write_baseline_table"]

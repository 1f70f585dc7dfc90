"""Driver layer: registry, script reader, device-resident NVE simulation."""

from .registry import RegistryError, StyleRegistry, resolve_style
from .script import ParseError, parse_script
from .simulation import (LJStyle, RunConfig, RunError, RunResult, Simulation, default_registry,
                         lattice_positions, run_script, seeded_velocities)

__all__ = ["RegistryError", "StyleRegistry", "resolve_style", "ParseError", "parse_script", "LJStyle", "RunConfig", "RunError",
           "RunResult", "Simulation", "default_registry", "lattice_positions", "run_script", "seeded_velocities"]

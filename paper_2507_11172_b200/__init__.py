"""B200-native (sm_100a) force-evaluation hot path for the arXiv 2507.11172
reference engine: Lennard-Jones + Axilrod-Teller-Muto forces with linked-cell
binning, integrated by r-RESPA multiple time-stepping.

Public names mirror the reference package ``respamd`` so the GPU path is a
drop-in: ``CudaLinkedCells`` for ``LinkedCells``, the functional passes, and a
device-resident ``respa_run``/``verlet_run``.  Importing this package does
not touch the GPU; the first pass loads ``librespa_b200.so`` and fails loudly
when the library or a CUDA device is missing.
"""

from .model import (CONTAINER_KINDS, ForceField, ParticleSystem, SamplingConfig, ScenarioConfig,
                    ValidationError, init_velocities, triplet_cutoff, wrap_positions)
from .grid import CellGrid
from .containers import (CudaDirectSum, CudaLinkedCells, MinimumSeparationError, build_cell_grid,
                         c01_pair_pass, c01_triplet_pass, collect_triplet_visits,
                         direct_sum_pairs, direct_sum_triplets, make_container, triplet_count)
from .integrators import IntegrationBlowUp, RespaSchedule, RunTrace, respa_run, verlet_run
from .scenarios import ExperimentPlan, ScenarioParseError, parse_scenario
from . import systems

__version__ = "0.1.0"

__all__ = [
    "CONTAINER_KINDS", "CellGrid", "CudaDirectSum", "CudaLinkedCells", "ExperimentPlan", "ForceField",
    "IntegrationBlowUp", "MinimumSeparationError", "ParticleSystem", "RespaSchedule", "RunTrace",
    "SamplingConfig", "ScenarioConfig", "ScenarioParseError", "ValidationError", "build_cell_grid",
    "c01_pair_pass", "c01_triplet_pass", "collect_triplet_visits", "direct_sum_pairs",
    "direct_sum_triplets", "init_velocities",
    "make_container", "parse_scenario", "respa_run", "systems", "triplet_count", "triplet_cutoff",
    "verlet_run", "wrap_positions",
]

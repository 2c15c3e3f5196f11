"""B200-native SPH density / smoothing-length pass -- a drop-in for the
reference package ``sphlab``'s hot path (density.py:286-413 of the
reference), built on hand-written sm_100a CUDA kernels behind a C ABI
(include/sph_b200.h, libsph_b200.so).

Public names mirror the reference's ``sphlab`` namespace for that path.
"""

from .checksum import density_checksum, fnv1a64
from .density import (
    DEFAULT_CHUNK_SIZE, DEFAULT_K, DEFAULT_MAX_ITERATIONS, H_GROWTH, PHASE_NAMES, PRESETS,
    ConvergenceError, DegenerateWorkloadError, LoopStyle, PassStats, SchedulerKind, SelectorKind,
    VariantConfig, adjust_smoothing_length, compute_density_pass, density_interact,
    density_pass_soa, initial_smoothing_length, preset_config,
)
from .kernel import WENDLAND_C6_NORM, KernelKind, KernelSpec, kernel_w
from .octree import DEFAULT_LEAF_CAPACITY, neighbor_counts, particle_perm
from .particles import (
    ALL_FIELDS, DEFAULT_AOS_RECORD_BYTES, DEFAULT_SCATTER_FIELDS, LIVE_RECORD_BYTES,
    SOA_MAX_BYTES_PER_PARTICLE, LayoutConfig, LayoutKind, ParticleSoA, aos_dtype, gather_to_soa,
    new_particle_array, scatter_from_soa,
)

__version__ = "0.1.0"

"""B200-native drop-in for the Modal Γ projection hot path (arXiv 1503.08809).

Python host layer over the C-ABI CUDA library (include/modal_b200.h).  The public names
mirror the reference package `cmbproj` for the two projection calls and their inputs:

    gamma3d_matrix(tables, mapping, grid, ...)      separable Γ  (cmbproj engine3d.py:156)
    gamma_nonsep(tables, mapping, grid, alpha, domain, ...)   non-separable sparse-grid path
    build_qtilde(inputs)                             stage 1: Δ_l(k), C_l, q̃ on the GPU

There is no CPU fallback: compute calls raise if the CUDA library or the GPU is missing.
"""

from .basis import (BasisTables, ModeMapping, RadialGrid, default_mode_mapping,
                    shifted_legendre)
from .engine3d import (DEFAULT_BLOCK, DomainRange, domain_count, domain_triples,
                       gamma3d_matrix, resolve_devices, triple_weights)
from .engine2d import PTable, build_ptable, gamma2d_matrix
from .gamma import GammaMatrix
from .gamma_io import (GammaFormatError, deserialize_gamma, load_checkpoint, merge_checkpoints,
                       save_checkpoint, serialize_gamma)
from .late_late import gamma_estimator, gamma_late_late
from .nonsep import SparseDomain, gamma_nonsep
from .plan import GammaPlan
from .qtilde import bessel_table, build_qtilde, build_qtilde_device
from .quadrature import (QuadratureRule, default_mu_points, gauss_legendre, integration_weights,
                         legendre_table, x_weights)
from .scheduler import ChunkPlan, make_plan, merge_partials, slab_plan

__version__ = "0.1.0"

__all__ = [
    "BasisTables", "ModeMapping", "RadialGrid", "default_mode_mapping", "shifted_legendre",
    "DEFAULT_BLOCK", "DomainRange", "domain_count", "domain_triples", "gamma3d_matrix",
    "resolve_devices",
    "triple_weights", "GammaMatrix", "SparseDomain", "gamma_nonsep", "GammaPlan",
    "bessel_table", "build_qtilde", "build_qtilde_device", "integration_weights", "x_weights",
    "ChunkPlan", "make_plan", "merge_partials", "slab_plan", "GammaFormatError",
    "serialize_gamma", "deserialize_gamma", "save_checkpoint", "load_checkpoint",
    "merge_checkpoints", "gamma_late_late", "gamma_estimator", "PTable", "build_ptable",
    "gamma2d_matrix", "QuadratureRule", "default_mu_points", "gauss_legendre",
    "legendre_table",
]

"""paper_2411_18889_b200 -- B200-native drop-in for the offloaded kernels of arXiv 2411.18889.

The reference (Solomon / ``pragmaport``) demonstrates its offload macros on
two kernels (pkg/tests/fixtures/listing_*.c).
This package is those kernels rebuilt for sm_100a behind their original
signatures:

* ``calc_acc(Ni, ipos, iacc, Nj, jpos, eps)``               -- listing_nbody.c:1
* ``diffusion3d(nx, ny, nz, dx, dy, dz, dt, kappa, f, fn)`` -- listing_diffusion.c:5

plus what the north star adds: the leapfrog KDK integrator, Plummer /
uniform particle setup, grid setup, and the multi-GPU partitioning in
``distributed``. All compute goes through ``lib/libsolomon_b200.so``
(include/solomon_b200.h); there is no CPU fallback.
"""
from ._lib import SolomonError, load  # noqa: F401
from .checkpoint import load as load_checkpoint, save as save_checkpoint  # noqa: F401
from .diffusion import Diffusion3D, coefficients, diffusion3d, diffusion3d_slab, init_grid  # noqa: F401
from .nbody import (  # noqa: F401
    Leapfrog,
    accelerations,
    calc_acc,
    energy,
    kdk_update,
    leapfrog_kdk,
    plummer,
    plummer_numpy,
    uniform,
    uniform_numpy,
    workspace,
)

__version__ = "0.1.0"

"""CPU oracle for the hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (and ``bench.py --impl reference``) may import this package. The product
package ``paper_2411_18889_b200`` never imports it and has no CPU fallback.

Two implementations live here:
  * ``Restatement`` -- ``solomon_oracle.c``: our operation-for-operation C
    restatement of the reference listings (plus the KDK spec, which has no
    reference counterpart).
  * ``Reference``   -- ``_ref/libref_*.so``: the reference's OWN listings,
    lowered by its transpiler's fallback backend and compiled with g++
    (``build_ref.py``). Parity is pinned against this build and against the
    golden vectors it produced (``tests/golden/``).
"""
from .loader import Reference, Restatement, cpu_isa, diffusion_coeffs  # noqa: F401

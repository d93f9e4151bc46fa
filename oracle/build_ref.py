"""Build ``oracle/_ref``: the reference's OWN CPU path for the hot path, compiled here.

TEST INFRASTRUCTURE ONLY -- nothing in ``paper_2411_18889_b200`` imports or links
this. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (and ``--impl reference``) use the result.

Recipe:
  1. Lower the paper's two listings with the reference transpiler's ``fallback``
     backend (host OpenMP) -- ``pragmaport.transpile`` (reference
     ``pkg/src/pragmaport/rewriter.py:29``) with ``Backend.FALLBACK``
     (``pkg/src/pragmaport/backends.py:15``), exactly what
     ``pragmaport transpile --backend fallback`` does (``cli.py:112-133``).
     Inputs: ``pkg/tests/fixtures/listing_nbody.c`` and ``listing_diffusion.c``.
  2. The generated ``.cpp`` files land in ``oracle/_ref/`` (git-ignored; they are
     generated from reference sources and never committed).
  3. ``oracle/ref_shim.cpp`` (ours) supplies the prelude the listings assume
     (``float4``, ``restrict``, ``<cmath>``) and ``extern "C"`` entry points.
  4. g++ builds two variants:
       libref_ieee.so  -O3 -march=<isa> -fopenmp   (IEEE; parity checker)
       libref_fast.so  -Ofast -march=<isa> -fopenmp (timing; mirrors PAPER.md:450,514)
     for <isa> in {native, x86-64-v3}; the loader picks by CPU flags.

Run only where ``/root/reference`` exists (this container). The built ``.so``
files travel to the GPU box inside the repo snapshot.
"""
from __future__ import annotations

import os
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
REF_ROOT = pathlib.Path(os.environ.get("SOLOMON_REFERENCE", "/root/reference"))
OUT = HERE / "_ref"

FIXTURES = {
    "nbody_fallback.cpp": "pkg/tests/fixtures/listing_nbody.c",
    "diffusion_fallback.cpp": "pkg/tests/fixtures/listing_diffusion.c",
}

VARIANTS = {
    # name: extra flags
    "ieee": ["-O3"],
    "fast": ["-Ofast"],
}
ISAS = {"native": "-march=native", "v3": "-march=x86-64-v3"}


def transpile_fixtures() -> None:
    sys.path.insert(0, str(REF_ROOT / "pkg" / "src"))
    try:
        from pragmaport import Backend, TranspileConfig, default_registry, transpile
    finally:
        sys.path.pop(0)
    reg = default_registry()
    OUT.mkdir(parents=True, exist_ok=True)
    for out_name, rel in FIXTURES.items():
        src = (REF_ROOT / rel).read_text()
        res = transpile(src, TranspileConfig(backend=Backend.FALLBACK), reg)
        text = f"// GENERATED from {rel} by pragmaport --backend fallback. Do not commit.\n" + res.text
        (OUT / out_name).write_text(text)


def compile_variants() -> list[pathlib.Path]:
    built = []
    shim = HERE / "ref_shim.cpp"
    for vname, vflags in VARIANTS.items():
        for iname, iflag in ISAS.items():
            so = OUT / f"libref_{vname}_{iname}.so"
            cmd = ["g++", "-std=c++17", *vflags, iflag, "-fopenmp", "-shared", "-fPIC",
                   f"-I{OUT}", str(shim), "-o", str(so)]
            subprocess.run(cmd, check=True)
            built.append(so)
    return built


def main() -> int:
    if not (REF_ROOT / "pkg").is_dir():
        print(f"build_ref: {REF_ROOT} not present; keeping prebuilt oracle/_ref", file=sys.stderr)
        return 0
    transpile_fixtures()
    for so in compile_variants():
        print(f"built {so.relative_to(HERE.parent)}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

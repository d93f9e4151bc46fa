"""Regenerate profiles/ncu_summary.json from `ncu --page raw --csv` exports.

    python scripts/ncu_summary.py profiles/r01/prof_force_r01d_raw.csv profiles/r01/prof_diff_r01d_raw.csv

bench.py reads ``dram_bytes_per_launch`` from it for the roofline ``traffic`` key.
"""
import csv
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
KEEP = {
    "k_force_fast": ["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                     "smsp__issue_active.avg.pct_of_peak_sustained_active",
                     "sm__warps_active.avg.pct_of_peak_sustained_active"],
    "k_diffusion_march": ["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                          "sm__warps_active.avg.pct_of_peak_sustained_active",
                          "smsp__issue_active.avg.pct_of_peak_sustained_active"],
    "k_diffusion_tb2": ["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                        "smsp__issue_active.avg.pct_of_peak_sustained_active",
                        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"],
    "k_leapfrog_small": ["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                         "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                         "smsp__issue_active.avg.pct_of_peak_sustained_active",
                         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"],
    "k_diffusion_resident": ["smsp__issue_active.avg.pct_of_peak_sustained_active",
                             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                             "lts__throughput.avg.pct_of_peak_sustained_elapsed"],
}
NOTES = {
    "k_force_fast": "N=2^20, 64 j-chunks reduced in-kernel in order (L2 ring, lines discarded): DRAM traffic ~ the 16 MiB in + 16 MiB out; FP32-pipe (register-file) bound",
    "k_diffusion_march": "512^3 step under ncu replay (cold L2); algorithmic 1.074 GB (8 B/cell)",
    "k_diffusion_tb2": "512^3, one launch = two steps, under ncu replay; algorithmic 1.074 GB (8 B/cell per launch)",
    "k_leapfrog_small": "BASELINE configs[0]: N=4096, all 16 KDK steps in one persistent launch (147 CTAs x 8 warps x 7 packed pairs, 128 j-chunks); the step-to-step exchange (arrival counters, bulk-copied slices, in-order reduce) is ~30% of a step",
    "k_diffusion_resident": "BASELINE configs[1]: 128^3 x 100 steps in one persistent launch (shared-memory-resident bricks); latency-bound per-step face exchange",
}


def num(s: str) -> float:
    return float(s.replace(",", ""))


def scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
            "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)


def summarise(path: pathlib.Path) -> tuple[str, dict]:
    rows = list(csv.reader(path.open()))
    hdr, units, row = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    name = row[col["Kernel Name"]]
    kernel = next(k for k in KEEP if k in name)
    get = lambda m: num(row[col[m]]) * scale(units[col[m]])  # noqa: E731
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out = {"dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
           "duration_s": get("gpu__time_duration.sum"),
           "registers": int(num(row[col["launch__registers_per_thread"]])),
           "grid": int(num(row[col["launch__grid_size"]])), "block": int(num(row[col["launch__block_size"]])),
           "source": str(path.relative_to(ROOT))}
    for m in KEEP[kernel]:
        if m in col:
            out[m] = num(row[col[m]])
    out["note"] = NOTES[kernel]
    return kernel, out


if __name__ == "__main__":
    summary = {}
    for p in sys.argv[1:]:
        k, v = summarise(pathlib.Path(p).resolve())
        summary[k] = v
    dst = ROOT / "profiles" / "ncu_summary.json"
    dst.write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps(summary, indent=1))

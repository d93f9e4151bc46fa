#!/usr/bin/env python
"""Benchmark: N-body Ginteractions/s & diffusion GLUPS on B200 vs roofline (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Prints ONE JSON line (rank 0). Headline = N-body (BASELINE configs[2] at
N=1: N=2^20 Plummer, one KDK step = one force evaluation + the fused
kick/drift; configs[3] for N>1: N=2^22 sharded over N GPUs with an NCCL
position all-gather). The diffusion numbers (configs[1]'s kernel at the
north star's 512^3 on one GPU; configs[4]'s 1024^3 slabs for N>1) ride in
``secondary.diffusion`` with their own roofline / cpu_baseline / e2e.

``--impl reference`` times the reference's OWN CPU implementation
(oracle/_ref: the paper's listings lowered by the reference transpiler's
fallback backend, g++ -Ofast -fopenmp) on the host cores, on bounded samples
of the same workloads. That leg and the ``cpu_baseline`` leg are the only
places this script touches ``oracle/``.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "N-body Ginteractions/s & diffusion GLUPS at 1/2/4/8 B200 vs roofline"
EPS = 2.0 ** -6
DT = 2.0 ** -7
FLOP_PER_INTERACTION = 20  # north-star convention
BYTES_PER_CELL = 8         # one read of f, one write of fn


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--particles", "--n", dest="n", type=int, default=None,
                    help="override particle count (use --particles under torchrun: --n clashes with its options)")
    ap.add_argument("--grid", type=int, default=None, help="override diffusion grid edge")
    ap.add_argument("--dsteps", type=int, default=50, help="timed diffusion steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-diffusion", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE parity configs [0] and [1]")
    ap.add_argument("--results", default=None,
                    help="also append the JSON line to this JSON-lines results file (rank 0)")
    ap.add_argument("--transport", choices=["auto", "p2p", "nccl"], default="auto",
                    help="N>1 data exchange: p2p = fused peer memory (position publish inside the update kernel; "
                         "edge-plane kernel pushing halo rows into the neighbours' mailboxes), nccl = collectives. "
                         "auto: p2p for both (falls back to nccl if peer mapping fails on any rank)")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU drivers (NCCL) even at world size 1 (smoke-tests the N>1 path)")
    ap.add_argument("--same-device", action="store_true",
                    help="test only: every rank on cuda:0 (gloo control plane, p2p transport) -- exercises the "
                         "N>1 bench path on a one-GPU box; the numbers are not a scaling measurement")
    ap.add_argument("--cpu-seconds", type=float, default=8.0, help="target CPU time per baseline sample")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md recipe)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=self.file, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.file.flush()
        rows = []
        for line in pathlib.Path(self.file.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.file.name)
        if not rows:
            return None
        reasons = sorted({self.NAMES[k] for _, _, r in rows for k in range(4) if r[k].lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "_source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(kernel: str):
    """dram bytes per launch for `kernel` from the committed ncu summary, or None."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel, {}).get("dram_bytes_per_launch")
    except (ValueError, AttributeError):
        return None


# ---------------------------------------------------------------------------
# CPU legs (the only users of oracle/)

def _omp_env():
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    os.environ.setdefault("OMP_PROC_BIND", "close")


def cpu_nbody_sample(pos, target_s: float, variant: str = "fast"):
    """Reference fallback build (-Ofast, or the IEEE -O3 build) on a bounded i-sample against all j.
    Returns (Ginter/s, ni, seconds)."""
    import numpy as np

    import oracle

    ref = oracle.Reference(variant)
    n = pos.shape[0]
    rng = np.random.default_rng(1234)
    t0 = time.perf_counter()
    probe = pos[rng.choice(n, 256, replace=False)]
    ref.calc_acc(probe, pos, EPS)
    dt0 = max(time.perf_counter() - t0, 1e-4)
    ni = int(min(n, max(256, 256 * target_s / dt0)))
    ni = max(64, ni // 64 * 64)
    sample = pos[rng.choice(n, ni, replace=False)]
    t0 = time.perf_counter()
    ref.calc_acc(sample, pos, EPS)
    dt = time.perf_counter() - t0
    return ni * n / dt / 1e9, ni, dt


def cpu_diffusion_sample(f_host, args, target_s: float, variant: str = "fast"):
    import oracle

    ref = oracle.Reference(variant)
    t0 = time.perf_counter()
    a = ref.diffusion3d(f_host, *args)
    dt0 = max(time.perf_counter() - t0, 1e-4)
    steps = int(max(1, min(50, target_s / dt0)))
    t0 = time.perf_counter()
    for _ in range(steps):
        a = ref.diffusion3d(a, *args)
    dt = time.perf_counter() - t0
    return f_host.size * steps / dt / 1e9, steps, dt


def cpu_info() -> str:
    try:
        for line in pathlib.Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def nbody_sample_parity(pos_np, acc_np, n_sample: int = 512, what: str = "the e2e drop-in output"):
    """Checker (oracle/_ref, the reference listing built -O3): a random i-sample of a full-size
    force evaluation against all j. SURVEY §8d tolerance for N = 2^20: relL2 <= 1e-4."""
    import numpy as np

    import oracle

    n = pos_np.shape[0]
    idx = np.sort(np.random.default_rng(1234).choice(n, n_sample, replace=False))
    want = oracle.Reference("ieee").calc_acc(np.ascontiguousarray(pos_np[idx]), pos_np, EPS)
    got = acc_np[idx]
    rel = float(np.linalg.norm(got[:, :3] - want[:, :3]) / np.linalg.norm(want[:, :3]))
    return {"relL2_acc": rel, "tolerance": 1e-4, "ok": rel <= 1e-4,
            "sample": f"{n_sample} random i x {n} j of {what} vs oracle/_ref libref_ieee"}


def diffusion_parity(f0, got, steps, dargs):
    """Checker: `steps` steps of the reference listing (oracle/_ref, -O3 IEEE build) vs the GPU field."""
    import numpy as np

    import oracle

    ref = oracle.Reference("ieee")
    want = ref.diffusion3d(f0, *dargs) if steps == 1 else ref.diffusion_run(f0, steps, *dargs)
    same = bool(np.array_equal(want.view(np.uint32), got.view(np.uint32)))
    return {"bit_identical": same, "steps": steps, "checker": "oracle/_ref libref_ieee",
            **({} if same else {"relL2": float(np.linalg.norm(got - want) / np.linalg.norm(want))})}


# ---------------------------------------------------------------------------
# reference arm

def run_reference(args, rank: int, world: int):
    if rank != 0:
        return None
    _omp_env()
    import numpy as np

    from paper_2411_18889_b200.nbody import plummer_numpy

    n = args.n or (1 << 20)
    pos, _ = plummer_numpy(n, 42)
    per_step = max(1.0, args.cpu_seconds / 2)
    for _ in range(args.warmup):
        cpu_nbody_sample(pos, per_step / 4)
    vals, nis = [], []
    t_all = 0.0
    for _ in range(args.steps):
        v, ni, dt = cpu_nbody_sample(pos, per_step)
        vals.append(v)
        nis.append(ni)
        t_all += dt
    value = statistics.mean(vals)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Ginteractions/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic Plummer sphere (seed 42)",
        "config": {"workload": f"nbody N={n} Plummer FP32 force evaluation (reference CPU: sampled i x all j)",
                   "n": n, "sample_i": nis[-1]},
        "cpu_baseline": {"value": value, "unit": "Ginteractions/s", "cores": cores, "kind": "reference",
                         "sample": f"{nis[-1]} random i x {n} j per step, libref_fast (g++ -Ofast -fopenmp), "
                                   f"{cpu_info()}"},
        "e2e": {"value": value, "unit": "Ginteractions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_diffusion:
        g = args.grid or 512
        f = np.random.default_rng(7).random((g, g, g), dtype=np.float32)
        dx = 1.0 / g
        dargs = (dx, dx, dx, 0.1 * dx * dx, 1.0)
        v, steps, dt = cpu_diffusion_sample(f, dargs, args.cpu_seconds)
        out["secondary"] = {"diffusion": {
            "metric": "diffusion GLUPS", "value": v, "unit": "GLUPS",
            "config": {"workload": f"diffusion3d {g}^3 FP32, {steps} steps (reference CPU)"},
            "cpu_baseline": {"value": v, "unit": "GLUPS", "cores": cores, "kind": "reference",
                             "sample": f"{steps} steps of {g}^3, libref_fast"}}}
    return out


# ---------------------------------------------------------------------------
# our arm

def run_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200 import _lib
    from paper_2411_18889_b200.distributed import ShardedLeapfrog, SlabDiffusion

    dev = torch.device("cuda", 0 if args.same_device else local_rank)
    if args.same_device:
        args.transport = "p2p"  # NCCL refuses two ranks on one GPU
    torch.cuda.set_device(dev)
    lib = b2.load()
    peaks = measured_peaks()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.same_device else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # FP32 roofline denominator, measured live on this GPU (MEASURED_PEAKS.json has no FP32 figure)
    probe = ctypes.CDLL(str(ROOT / "paper_2411_18889_b200" / "lib" / "libsolomon_probe.so"))
    probe.solomon_probe_fp32_tflops.restype = ctypes.c_double
    fp32_peak = probe.solomon_probe_fp32_tflops(5)
    fp32_source = ("measured live: packed-FFMA2 throughput probe on this GPU "
                   "(nominal 148x128x2x1.965 GHz = 74.4)")
    for k, v in peaks.items():  # a driver-measured FP32 figure, if MEASURED_PEAKS.json carries one, wins
        if "fp32" in k.lower() and isinstance(v, (int, float)) and 20.0 < float(v) < 200.0:
            fp32_peak, fp32_source = float(v), f"MEASURED_PEAKS.json {k}"
            break

    # ---------------- N-body ----------------
    sharded = world > 1 or args.dist
    n = args.n or ((1 << 20) if world == 1 else (1 << 22))
    pos_np, vel_np = b2.plummer_numpy(n, 42)
    if not sharded:
        pos = torch.from_numpy(pos_np).to(dev)
        vel = torch.from_numpy(vel_np).to(dev)
        nch = lib.b2_calc_acc_nchunks(n, 0)
        part = torch.empty((nch * n, 4), dtype=torch.float32, device=dev)
        acc = torch.empty_like(pos)
        h = 0.5 * DT
        sh = _lib.stream_handle(dev)

        def force():
            _lib.check(lib.b2_calc_acc_partials(n, pos.data_ptr(), n, pos.data_ptr(), EPS, 0, part.data_ptr(), sh),
                       "partials")

        def update(phases):
            _lib.check(lib.b2_kdk_update(n, pos.data_ptr(), vel.data_ptr(), acc.data_ptr(), part.data_ptr(), nch,
                                         h, h, DT, phases, sh), "update")

        force()
        update(_lib.B2_KDK_REDUCE)
        update(_lib.B2_KDK_KICK_DRIFT)
        steady = _lib.B2_KDK_REDUCE | _lib.B2_KDK_KICK_END | _lib.B2_KDK_KICK_DRIFT

        def step(evs):
            evs[0].record(stream)
            force()
            evs[1].record(stream)
            update(steady)
            evs[2].record(stream)

        n_local = n
        launches_per_step = 2
        parallelism = "single GPU"
    else:
        plan_lo = rank * (n // world)
        nb_transport = "p2p" if args.transport == "auto" else args.transport
        try:
            sim = ShardedLeapfrog(torch.from_numpy(pos_np[plan_lo:plan_lo + n // world]).to(dev),
                                  torch.from_numpy(vel_np[plan_lo:plan_lo + n // world]).to(dev), EPS, DT,
                                  transport=nb_transport)
        except Exception as e:  # noqa: BLE001
            print(f"p2p position transport unavailable ({e}); using NCCL", file=sys.stderr)
            nb_transport = "nccl"
            sim = ShardedLeapfrog(torch.from_numpy(pos_np[plan_lo:plan_lo + n // world]).to(dev),
                                  torch.from_numpy(vel_np[plan_lo:plan_lo + n // world]).to(dev), EPS, DT,
                                  transport=nb_transport)
        sim.step(1, close=False)
        n_local = n // world
        steady = _lib.B2_KDK_REDUCE | _lib.B2_KDK_KICK_END | _lib.B2_KDK_KICK_DRIFT

        def step(evs):
            hh = 0.5 * DT
            evs[0].record(stream)
            if nb_transport == "nccl":
                sim.gather()
            else:
                sim._await_peers()
            evs[3].record(stream)
            sim.k.partials(sim.pos, sim.pos_all, sim.eps, sim.part)
            evs[1].record(stream)
            if nb_transport == "nccl":
                sim.k.update(sim.pos, sim.vel, sim.acc, sim.part, sim.nch, hh, hh, DT, steady)
            else:
                sim._publish_update(sim.vel, sim.part, hh, hh, DT, steady)
            evs[2].record(stream)

        launches_per_step = 2
        parallelism = (f"i-shard x{world}, " + ("NCCL all_gather_into_tensor of positions per step"
                                                  if nb_transport == "nccl" else
                                                  "positions published to every peer by the update kernel "
                                                  "(fused all-gather over peer memory)"))

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(4)]  # noqa: E731
    for _ in range(args.warmup):
        flush.zero_()
        step(mk())
    torch.cuda.synchronize(dev)
    barrier()
    clocks = ClockSampler(dev.index).start() if rank == 0 else None
    torch.cuda.synchronize(dev)
    barrier()
    events = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        evs = mk()
        step(evs)
        events.append(evs)
    torch.cuda.synchronize(dev)
    barrier()
    clock_rec = clocks.stop() if clocks else None
    step_ms = [e[0].elapsed_time(e[2]) for e in events]
    force_ms = [(e[3] if sharded else e[0]).elapsed_time(e[1]) for e in events]
    total_ms = max_over_ranks(sum(step_ms))
    force_avg = max_over_ranks(statistics.mean(force_ms))
    gather_ms = max_over_ranks(statistics.mean(e[0].elapsed_time(e[3]) for e in events)) if sharded else 0.0
    interactions = float(n) * float(n)
    value = interactions * args.steps / (total_ms * 1e-3) / 1e9
    achieved_tf = FLOP_PER_INTERACTION * float(n_local) * float(n) / (force_avg * 1e-3) / 1e12

    result = {
        "metric": METRIC, "value": value, "unit": "Ginteractions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: Plummer sphere (seed 42, FP64 -> FP32 on host); diffusion grid U[0,1) (seed 7)",
        "config": {
            "workload": (f"nbody N={n} Plummer FP32, one KDK leapfrog step per step "
                         f"(force evaluation of N^2 interactions + fused reduce/kick/drift)"),
            "n": n, "eps": EPS, "dt": DT, "jchunks": int(lib.b2_calc_acc_nchunks(n, 0)),
            "parallelism": parallelism,
            "l2": "flushed between timed steps (512 MiB memset, outside the step events)",
        },
        "roofline": {
            "bound": "fp32", "kernel": "k_force_fast", "achieved": achieved_tf, "peak": fp32_peak,
            "unit": "TFLOP/s", "frac": achieved_tf / fp32_peak if fp32_peak > 0 else None,
            "traffic": ncu_traffic("k_force_fast"),
            "traffic_note": ("DRAM bytes per launch (ncu --set full): almost all of it is the write of the "
                             "64 j-chunk partial sums (N x 64 x 16 B) that the update kernel reduces in a fixed "
                             "order; ~0.2 ms of HBM time in a ~400 ms FP32-bound launch"),
            "flop_per_interaction": FLOP_PER_INTERACTION,
            "peak_source": fp32_source,
            "force_ms": force_avg, "allgather_ms": gather_ms,
        },
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clock_rec,
    }

    # e2e through the reference-facing drop-in with HOST (pinned) buffers
    if world == 1:
        hpos = torch.from_numpy(pos_np).pin_memory()
        hacc = torch.empty_like(hpos).pin_memory()
        P = ctypes.c_void_p
        lib.calc_acc(n, P(hpos.data_ptr()), P(hacc.data_ptr()), n, P(hpos.data_ptr()), EPS)  # warm the arena
        t0 = time.perf_counter()
        k_e2e = max(1, min(args.steps, 3))
        for _ in range(k_e2e):
            lib.calc_acc(n, P(hpos.data_ptr()), P(hacc.data_ptr()), n, P(hpos.data_ptr()), EPS)
        t_e2e = (time.perf_counter() - t0) / k_e2e
        _lib.check(lib.b2_last_error(), "calc_acc drop-in")
        if rank == 0 and not args.no_cpu_baseline:
            try:
                result["parity"] = nbody_sample_parity(pos_np, hacc.numpy())
            except FileNotFoundError as e:
                result["parity"] = {"unavailable": str(e)}
        result["e2e"] = {"value": interactions / t_e2e / 1e9, "unit": "Ginteractions/s",
                         "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                         "api": "calc_acc(Ni, ipos, iacc, Nj, jpos, eps) C drop-in, pinned host buffers "
                                "(ipos == jpos staged once), synchronous", "steps": k_e2e}
        del hpos, hacc
    else:
        # e2e through the public driver API with HOST buffers: every step copies this rank's
        # positions in from pinned memory, runs ShardedLeapfrog.step (exchange + force + update)
        # and reads its accelerations back; wall time, max over ranks
        hpos = sim.pos.cpu().pin_memory()
        hacc = torch.empty_like(hpos).pin_memory()
        k_e2e = max(1, min(args.steps, 2))
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            sim.pos.copy_(hpos, non_blocking=True)
            sim.step(1, close=False)
            hacc.copy_(sim.acc, non_blocking=True)
        torch.cuda.synchronize(dev)
        t_e2e = max_over_ranks(time.perf_counter() - t0) / k_e2e
        result["e2e"] = {"value": interactions / t_e2e / 1e9, "unit": "Ginteractions/s",
                         "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                         "api": "ShardedLeapfrog.step(1) per step with each rank's positions copied in from "
                                "pinned host memory and its accelerations read back (whole-job bytes)",
                         "steps": k_e2e}
        del hpos, hacc
        # parity at the sharded size: every rank publishes its positions, rank 0 checks a sample of
        # a device force evaluation over the gathered pos_all against the reference build
        sim.gather()
        torch.cuda.synchronize(dev)
        barrier()
        if rank == 0 and not args.no_cpu_baseline:
            import paper_2411_18889_b200 as b2

            allpos = sim.pos_all.contiguous()
            out = torch.empty_like(allpos)
            b2.calc_acc(n, allpos, out, n, allpos, EPS)
            try:
                result["parity"] = nbody_sample_parity(allpos.cpu().numpy(), out.cpu().numpy(),
                                                       what="calc_acc on rank 0 over pos_all after the sharded run")
            except FileNotFoundError as e:
                result["parity"] = {"unavailable": str(e)}
        barrier()

    # ---------------- diffusion ----------------
    if not args.no_diffusion:
        result["secondary"] = {"diffusion": run_diffusion(args, rank, world, dev, stream, peaks, barrier,
                                                          max_over_ranks, flush)}

    if world == 1 and not args.no_configs:
        try:
            result["parity_configs"] = run_parity_configs(dev)
        except FileNotFoundError as e:
            result["parity_configs"] = {"unavailable": str(e)}

    # ---------------- CPU baseline (rank 0, N=1) ----------------
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        _omp_env()
        cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
        try:
            v, ni, dt = cpu_nbody_sample(pos_np, args.cpu_seconds)
            result["cpu_baseline"] = {"value": v, "unit": "Ginteractions/s", "cores": cores, "kind": "reference",
                                      "sample": f"{ni} random i x {n} j (one sampled force evaluation, {dt:.1f} s), "
                                                f"oracle/_ref libref_fast (reference listing via its fallback "
                                                f"lowering, g++ -Ofast -fopenmp), {cpu_info()}"}
            v3, ni3, dt3 = cpu_nbody_sample(pos_np, args.cpu_seconds / 3, "ieee")
            result["cpu_baseline"]["ieee"] = {"value": v3, "sample": f"{ni3} random i x {n} j ({dt3:.1f} s), "
                                                                     "oracle/_ref libref_ieee (g++ -O3 -fopenmp)"}
        except FileNotFoundError as e:
            result["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    return result


def run_diffusion(args, rank, world, dev, stream, peaks, barrier, max_over_ranks, flush):
    import torch

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import SlabDiffusion

    lib = b2.load()
    g = args.grid or (512 if world == 1 else 1024)
    dx = 1.0 / g
    dargs = (dx, dx, dx, 0.1 * dx * dx, 1.0)
    single = world == 1 and not args.dist
    transport = None
    if single:
        f = b2.init_grid(g, g, g, seed=7, device=dev)
        fn = torch.empty_like(f)
        bufs = [f, fn]

        def dstep(i):
            a, b = bufs[i % 2], bufs[(i + 1) % 2]
            b2.diffusion3d(g, g, g, *dargs, a, b)

        launches = 1
        nxl = g
    else:
        nxl = g // world
        gen = torch.Generator(device=dev).manual_seed(7 + rank)
        f_local = torch.rand((nxl, g, g), generator=gen, dtype=torch.float32, device=dev)
        transport = "p2p" if args.transport == "auto" else args.transport
        try:
            sim = SlabDiffusion(f_local, *dargs, transport=transport)
        except Exception as e:  # noqa: BLE001 -- report and fall back to the NCCL transport
            print(f"p2p halo transport unavailable ({e}); using NCCL", file=sys.stderr)
            transport = "nccl"
            sim = SlabDiffusion(f_local, *dargs, transport=transport)

        def dstep(i):
            sim.step(1)

        launches = sim.launches_per_step()
    for i in range(5):
        dstep(i)
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.dsteps):  # back to back: inputs (2 x field) exceed L2, no flush needed
        dstep(i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    total_ms = max_over_ranks(e0.elapsed_time(e1))
    step_ms = total_ms / args.dsteps
    cells = float(g) ** 3
    glups = cells * args.dsteps / (total_ms * 1e-3) / 1e9
    kernel_ms = step_ms  # one launch per step at N=1: average launch duration over the timed region
    achieved = BYTES_PER_CELL * float(nxl) * g * g / (kernel_ms * 1e-3) / 1e9
    out = {
        "metric": "diffusion GLUPS", "value": glups, "unit": "GLUPS", "ms_per_step": step_ms,
        "steps": args.dsteps, "warmup": 5, "dtype": "f32",
        "config": {"workload": f"diffusion3d {g}^3 FP32 7-point step" + (
                       " (single GPU)" if single else f", i-slabs x{world}, halo transport {transport}"),
                   "grid": [g, g, g], "dt_over_dx2": 0.1,
                   "l2": "inputs (2 x {:.0f} MiB per GPU) larger than L2; no flush".format(4 * nxl * g * g / 2**20)},
        "roofline": {"bound": "hbm", "kernel": "k_diffusion_march", "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                     "traffic": ncu_traffic("k_diffusion_march"), "bytes_per_cell": BYTES_PER_CELL,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_source" not in peaks else peaks["_source"]},
        "gpu_launches": launches * args.dsteps,
    }
    if not single:
        out["parity"] = slab_parity(sim, rank, world, dev, dargs, args)
        out["run"] = run_slab_multistep(sim, args, rank, world, dev, stream, peaks, g, nxl, barrier, max_over_ranks,
                                        dargs)
    if single:
        host_f = f.cpu().pin_memory()
        host_fn = torch.empty_like(host_f).pin_memory()
        P = ctypes.c_void_p
        lib.diffusion3d(g, g, g, *dargs, P(host_f.data_ptr()), P(host_fn.data_ptr()))
        k = 3
        t0 = time.perf_counter()
        for _ in range(k):
            lib.diffusion3d(g, g, g, *dargs, P(host_f.data_ptr()), P(host_fn.data_ptr()))
        t = (time.perf_counter() - t0) / k
        if rank == 0 and not args.no_cpu_baseline:
            try:
                out["parity"] = diffusion_parity(host_f.numpy(), host_fn.numpy(), 1, dargs)
            except FileNotFoundError as e:
                out["parity"] = {"unavailable": str(e)}
        out["e2e"] = {"value": cells / t / 1e9, "unit": "GLUPS", "h2d_bytes_per_step": int(4 * cells),
                      "d2h_bytes_per_step": int(4 * cells),
                      "api": "diffusion3d(nx,...,f,fn) C drop-in, pinned host buffers, synchronous"}
        if rank == 0 and not args.no_cpu_baseline:
            _omp_env()
            try:
                v, steps, dt = cpu_diffusion_sample(host_f.numpy(), dargs, args.cpu_seconds / 2)
                out["cpu_baseline"] = {"value": v, "unit": "GLUPS",
                                       "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
                                       "kind": "reference",
                                       "sample": f"{steps} steps of {g}^3 ({dt:.1f} s), oracle/_ref libref_fast"}
                v3, steps3, dt3 = cpu_diffusion_sample(host_f.numpy(), dargs, args.cpu_seconds / 6, "ieee")
                out["cpu_baseline"]["ieee"] = {"value": v3, "sample": f"{steps3} steps of {g}^3 ({dt3:.1f} s), "
                                                                      "oracle/_ref libref_ieee (g++ -O3 -fopenmp)"}
            except FileNotFoundError as e:
                out["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        del host_f, host_fn
        out["run"] = run_diffusion_multistep(args, dev, stream, peaks, g, dargs)
    return out


def slab_parity(sim, rank, world, dev, dargs, args):
    """One more sharded step; rank 0 checks its slab bit for bit against the reference listing run
    on its planes plus rank 1's first plane (the only neighbour data its planes read)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    if args.no_cpu_baseline:
        return None
    on_dev = dist.get_backend() == "nccl"
    f0 = sim.f.clone() if rank == 0 else None
    nb = None
    if rank == 1 and world > 1:
        plane = sim.f[0].contiguous()
        dist.send(plane if on_dev else plane.cpu(), 0)
    elif rank == 0 and world > 1:
        nb = torch.empty(sim.f.shape[1:], dtype=sim.f.dtype, device=dev if on_dev else "cpu")
        dist.recv(nb, 1)
    sim.step(1)
    torch.cuda.synchronize(dev)
    if rank != 0:
        return None
    try:
        import oracle

        if world > 1:
            sub = np.concatenate([f0.cpu().numpy(), nb.cpu().numpy()[None]], axis=0)
            want = oracle.Reference("ieee").diffusion3d(sub, *dargs)[:-1]
        else:  # the slab is the whole grid
            want = oracle.Reference("ieee").diffusion3d(f0.cpu().numpy(), *dargs)
        got = sim.f.cpu().numpy()
        return {"bit_identical": bool(np.array_equal(want.view(np.uint32), got.view(np.uint32))), "steps": 1,
                "checker": "oracle/_ref libref_ieee on rank 0's planes + rank 1's first plane",
                "planes": int(got.shape[0])}
    except FileNotFoundError as e:
        return {"unavailable": str(e)}


def run_slab_multistep(sim, args, rank, world, dev, stream, peaks, g, nxl, barrier, max_over_ranks, dargs):
    """N > 1: SlabDiffusion.run -- two steps per exchange of two halo planes, each pass one
    b2_diffusion3d_run(..., 2) over the halo-extended slab (two steps per HBM pass on large
    slabs). Effective GLUPS = all cells x steps / time (max over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    steps = max(2, args.dsteps // 2 * 2)
    sim.run(4)
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sim.run(steps)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    cells = float(g) ** 3
    nx_ext = nxl + (2 if sim.has_lo else 0) + (2 if sim.has_hi else 0)
    pass_ms = 2 * ms / steps
    achieved = BYTES_PER_CELL * float(nx_ext) * g * g / (pass_ms * 1e-3) / 1e9
    out = {
        "metric": "diffusion GLUPS, multi-step sharded run (effective)", "value": cells * steps / (ms * 1e-3) / 1e9,
        "unit": "GLUPS", "ms_per_step": ms / steps, "steps": steps, "warmup": 4,
        "config": {"workload": f"SlabDiffusion.run({steps}) on {g}^3 FP32, i-slabs x{world}, two steps per "
                               f"exchange of two halo planes (transport {sim.transport})",
                   "grid": [g, g, g], "l2": "inputs larger than L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": "k_diffusion_tb2 (per rank, halo-extended slab)", "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                     "bytes_per_cell_per_launch": BYTES_PER_CELL, "steps_per_launch": 2},
        "gpu_launches": (steps // 2) * (3 if sim.transport == "p2p" and world > 1 else 1),
    }
    # parity: two more steps; rank 0 checks its planes against the reference listing run on
    # them plus rank 1's first two planes (the light cone of two steps)
    if args.no_cpu_baseline:
        return out
    on_dev = dist.get_backend() == "nccl"
    f0 = sim.f.clone() if rank == 0 else None
    nb = None
    if rank == 1:
        two = sim.f[0:2].contiguous()
        dist.send(two if on_dev else two.cpu(), 0)
    elif rank == 0 and world > 1:
        nb = torch.empty((2,) + tuple(sim.f.shape[1:]), dtype=sim.f.dtype, device=dev if on_dev else "cpu")
        dist.recv(nb, 1)
    sim.run(2)
    torch.cuda.synchronize(dev)
    if rank == 0:
        try:
            import oracle

            sub = f0.cpu().numpy() if nb is None else np.concatenate([f0.cpu().numpy(), nb.cpu().numpy()], axis=0)
            want = oracle.Reference("ieee").diffusion_run(sub, 2, *dargs)[:nxl]
            got = sim.f.cpu().numpy()
            out["parity"] = {"bit_identical": bool(np.array_equal(want.view(np.uint32), got.view(np.uint32))),
                             "steps": 2, "checker": "oracle/_ref libref_ieee on rank 0's planes + rank 1's first two"}
        except FileNotFoundError as e:
            out["parity"] = {"unavailable": str(e)}
    return out


def run_diffusion_multistep(args, dev, stream, peaks, g, dargs):
    """The device-resident time loop (Diffusion3D.run -> b2_diffusion3d_run): on large grids two
    steps per HBM pass (k_diffusion_tb2). Effective GLUPS = cells x steps / time."""
    import torch

    import paper_2411_18889_b200 as b2

    f0 = b2.init_grid(g, g, g, seed=7, device=dev)
    steps = max(2, args.dsteps // 2 * 2)
    sim = b2.Diffusion3D(f0.clone(), *dargs)
    sim.run(4)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sim.run(steps)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    cells = float(g) ** 3
    pass_ms = 2 * ms / steps  # one k_diffusion_tb2 launch = two steps
    achieved = BYTES_PER_CELL * cells / (pass_ms * 1e-3) / 1e9
    # end to end from host memory: pinned H2D of the field, the run, D2H of the result
    host = f0.cpu().pin_memory()
    back = torch.empty_like(host).pin_memory()
    sim2 = b2.Diffusion3D(torch.empty_like(f0), *dargs)  # device buffers allocated outside the timed region
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    sim2.f.copy_(host, non_blocking=True)
    sim2.run(steps)
    back.copy_(sim2.field, non_blocking=True)
    torch.cuda.synchronize(dev)
    t_e2e = time.perf_counter() - t0
    parity = None
    if not args.no_cpu_baseline:
        try:
            parity = diffusion_parity(host.numpy(), back.numpy(), steps, dargs)
        except FileNotFoundError as e:
            parity = {"unavailable": str(e)}
    return {
        "parity": parity,
        "metric": "diffusion GLUPS, multi-step device-resident run (effective)", "value": cells * steps / (ms * 1e-3) / 1e9,
        "unit": "GLUPS", "ms_per_step": ms / steps, "steps": steps, "warmup": 4,
        "config": {"workload": f"Diffusion3D.run({steps}) on {g}^3 FP32 (b2_diffusion3d_run: two steps per HBM pass)",
                   "grid": [g, g, g], "l2": "inputs (2 x field) larger than L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": "k_diffusion_tb2", "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": ncu_traffic("k_diffusion_tb2"),
                     "bytes_per_cell_per_launch": BYTES_PER_CELL, "steps_per_launch": 2},
        "gpu_launches": steps // 2,
        "e2e": {"value": cells * steps / t_e2e / 1e9, "unit": "GLUPS", "h2d_bytes_per_step": int(4 * cells / steps),
                "d2h_bytes_per_step": int(4 * cells / steps),
                "api": f"pinned host field -> Diffusion3D(...).run({steps}) -> pinned host (one copy each way per run)"},
    }


def run_parity_configs(dev):
    """BASELINE configs[0] and [1] (the CPU-reference-run parity cases): GPU time, CPU time, parity."""
    import numpy as np
    import torch

    import oracle
    import paper_2411_18889_b200 as b2

    _omp_env()
    out = {}
    # configs[0]: N=4096 Plummer FP32, 16 leapfrog steps
    n, eps, dt, steps = 4096, EPS, DT, 16
    pos, vel = b2.plummer_numpy(n, 42)
    lf = b2.Leapfrog(torch.from_numpy(pos).to(dev), torch.from_numpy(vel).to(dev), eps, dt)
    lf.step(2)
    lf = b2.Leapfrog(torch.from_numpy(pos).to(dev), torch.from_numpy(vel).to(dev), eps, dt)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lf.step(steps)
    e1.record()
    torch.cuda.synchronize(dev)
    gpu_ms = e0.elapsed_time(e1)
    rs = oracle.Restatement()
    t0 = time.perf_counter()
    wp, wv, wa = rs.leapfrog(pos, vel, eps, dt, steps)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    gp, gv = lf.pos.cpu().numpy(), lf.vel.cpu().numpy()
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    # physics check (the integrator has no reference): total energy drift over the 16 steps
    p0 = torch.from_numpy(pos).to(dev)
    e_start = sum(b2.energy(p0, torch.from_numpy(vel).to(dev), b2.accelerations(p0, eps, potential=True), eps))
    e_end = sum(b2.energy(lf.pos, lf.vel, b2.accelerations(lf.pos, eps, potential=True), eps))
    out["nbody_4096_plummer_kdk16"] = {
        "config": "BASELINE configs[0]: N=4096 Plummer FP32, 16 leapfrog steps",
        "gpu_ms": gpu_ms, "gpu_launches": 1,
        "path": "b2_leapfrog -> k_leapfrog_small (all 16 KDK steps in one persistent launch, positions "
                "exchanged between CTAs as tagged 16-byte words; + one memset), bit-identical to the "
                "two-kernel-per-step path",
        "gpu_ginteractions_per_s": n * n * steps / (gpu_ms * 1e-3) / 1e9,
        "cpu_ms": cpu_ms, "cpu_kind": "port (oracle/solomon_oracle.c KDK around the restated calc_acc; "
                                      "the reference has no integrator)",
        "cpu_cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
        "parity_relL2": {"pos": rel(gp[:, :3], wp[:, :3]), "vel": rel(gv[:, :3], wv[:, :3])},
        "tolerance": {"pos": 1e-5, "vel": 1e-4},
        "energy": {"start": e_start, "end": e_end, "rel_drift": abs(e_end - e_start) / abs(e_start)},
    }
    # configs[1]: 128^3 diffusion, 100 steps
    g, dsteps = 128, 100
    dx = 1.0 / g
    dargs = (dx, dx, dx, 0.1 * dx * dx, 1.0)
    f0 = b2.init_grid(g, g, g, seed=7, device=dev)
    sim = b2.Diffusion3D(f0.clone(), *dargs)
    sim.run(10)
    sim = b2.Diffusion3D(f0.clone(), *dargs)
    torch.cuda.synchronize(dev)
    e0.record()
    sim.run(dsteps)
    e1.record()
    torch.cuda.synchronize(dev)
    gpu_ms = e0.elapsed_time(e1)
    host = f0.cpu().numpy()
    ref = oracle.Reference("ieee")
    fast = oracle.Reference("fast")
    t0 = time.perf_counter()
    fast.diffusion_run(host, dsteps, *dargs)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    want = ref.diffusion_run(host, dsteps, *dargs)
    got = sim.field.cpu().numpy()
    out["diffusion_128_100steps"] = {
        "config": "BASELINE configs[1]: 128^3 grid, 100 steps, single B200 (L2-resident: 2 x 8 MiB)",
        "gpu_ms": gpu_ms, "gpu_launches": 1,
        "path": "b2_diffusion3d_run -> k_diffusion_resident (shared-memory-resident bricks, one persistent "
                "launch for all steps; + one memset of the face mailbox)",
        "gpu_glups": g ** 3 * dsteps / (gpu_ms * 1e-3) / 1e9,
        "cpu_ms": cpu_ms, "cpu_kind": "reference (oracle/_ref libref_fast)",
        "cpu_glups": g ** 3 * dsteps / (cpu_ms * 1e-3) / 1e9,
        "cpu_cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
        "parity": "bit-identical" if np.array_equal(got.view(np.uint32), want.view(np.uint32)) else
                  f"MISMATCH relL2 {rel(got, want):.3e}",
    }
    return out


def _claim_stdout():
    """stdout carries exactly one JSON line: keep a private handle on it and point fd 1 at stderr,
    so that native libraries writing to fd 1 (NCCL prints its version banner there) cannot add
    lines the driver would have to skip."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return out


def _emit(line: dict, json_out, results: str | None) -> None:
    text = json.dumps(line)
    print(text, file=json_out, flush=True)
    if results:
        with open(results, "a") as fh:
            fh.write(text + "\n")


def main():
    json_out = _claim_stdout()
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            _emit(out, json_out, args.results)
        return
    if world > 1 or args.dist:
        from paper_2411_18889_b200.distributed import init_distributed

        # a lost rank fails the run instead of hanging it
        init_distributed("gloo" if args.same_device else "nccl", timeout_s=900.0)
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        _emit(out, json_out, args.results)
    if world > 1 or args.dist:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

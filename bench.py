"""bench.py — inertia evaluations nu_sigma/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kep|reference] [--config 4]

Workload (BASELINE.json configs[3], "c4"): the n = 1,500,000 quasi-1D
tight-binding pencil (10 x 10 x 3750 atoms, 4 orbitals, periodic z, cutoff
1.8), synthetic and seeded (kepgen).  One STEP is
one multisection round of stage 2 (Alg. 1' generalised to P = N x S shifts per
round; paper_1710_05134_b200.multisection): every rank
factorises S = 16 shifts of the current bracket (one LDL^T of A - sigma B each,
rows a1-a5 of SURVEY.md §8), the int64 counts (and the shifts actually
evaluated) are all-gathered over NCCL and every rank applies the same bracket
update; a bracket holding <= m_max = 20 eigenvalues restarts from the initial
one.  Weak scaling: S shifts per GPU per step.

value = shifts factorised by all ranks / max-over-ranks device time of the K
timed steps (CUDA events on the library's stream, barrier + synchronize on
both sides).  e2e = the same through the public C-ABI call with HOST buffers:
every step uploads A and B values from pinned host memory (kep_set_values)
and reads the counts back.  The fronts (tens of GB) are far larger than L2,
so no L2 flush is needed between steps.  time_to_bracket = one complete
stage 2 from the initial interval to nu_u - nu_l <= m_max.

--gpus N without torchrun's environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1).

cpu_baseline / --impl reference: the CPU oracle (oracle.sparse_mf, O-sparse,
as it stands) on C = all host cores, one shift per worker process with one
BLAS thread (shift-parallel, like multisection), on a bounded sample of the
workload: the c4 recipe on a 10 x 10 x L periodic sub-wire.  Its measured
wall time is scaled to full-size c4 shifts by the ratio of the oracle's own
flop counts (tests/golden/oracle_flops.json, written by
scripts/oracle_flops.py); the scale and the unscaled numbers are reported.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

M_MAX = 20
METRIC = "inertia evals nu_sigma/sec (LDL^T of A - sigma B), n=1.5M"


def _clock_sampler(stop, out, device_index):
    cmd = ["nvidia-smi", "-i", str(device_index),
           "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
           "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
           "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"]
    try:
        pr = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except Exception:
        return
    while not stop.is_set():
        line = pr.stdout.readline()
        if not line:
            break
        out.append(line.strip())
    pr.terminate()


def _clock_summary(lines):
    sm, mx, reasons = [], None, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for ln in lines:
        f = [x.strip() for x in ln.split(",")]
        if len(f) < 7:
            continue
        try:
            sm.append(float(f[0]))
            mx = float(f[1])
        except ValueError:
            continue
        for nm, v in zip(names, f[3:7]):
            if v.lower().startswith("active"):
                reasons.add(nm)
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
            "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak_tflops():
    """cuBLAS DGEMM 8192^3 best of 5 (the FP64 roofline denominator, measured live:
    MEASURED_PEAKS.json has no FP64 entry)."""
    import torch
    N = 8192
    a = torch.randn(N, N, dtype=torch.float64, device="cuda")
    b = torch.randn(N, N, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b, c
    torch.cuda.empty_cache()
    return 2.0 * N ** 3 / best / 1e12


def workload_config(cfg: int, shape, world: int, S: int) -> dict:
    """The `config` object of the JSON line: the workload only, identical in both arms."""
    import kepgen
    kw = dict(kepgen.CONFIGS[cfg])
    shp = tuple(shape) if shape else kw["shape"]
    n = int(np.prod(shp)) * kw["o"]
    return {"workload": f"c{cfg}" + (f"-{'x'.join(map(str, shp))}" if shape else ""),
            "lattice": "x".join(map(str, shp)), "orbitals": kw["o"], "cutoff": kw["cutoff"],
            "periodic": list(kw["periodic"]), "seed": kw["seed"], "n": n,
            "shifts_per_gpu_per_step": S, "shifts_per_step": S * world,
            "l2": "inputs larger than L2 (fronts ~GBs per shift); no flush"}


# ----------------------------------------------------------------------------- CPU oracle (baseline / reference arm)
_SAMPLE = None


def _oracle_worker_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:                                    # pragma: no cover
        pass


def _oracle_worker(sigma):
    t = time.time()
    r = _SAMPLE.inertia(float(sigma))
    return time.time() - t, int(r.n_neg)


class OracleSample:
    """The oracle as it stands on a bounded sample of the workload (or, length=None, on the full
    workload itself), C worker processes."""

    def __init__(self, cfg: int, length, pencil=None, bounds=None):
        import kepgen
        from oracle.sparse_mf import SparseOracle
        global _SAMPLE
        if cfg != 4:
            raise ValueError("the CPU sample is defined for the c4 workload")
        base = kepgen.CONFIGS[cfg]["shape"]
        self.shape = tuple(base) if length is None else (base[0], base[1], length)
        p = pencil if (pencil is not None and length is None) else kepgen.config(cfg, shape=None if length is None else self.shape)
        self.n = p.n
        _SAMPLE = SparseOracle(p)
        lo, hi = bounds if (bounds is not None and length is None) else kepgen.spectral_bounds(p)
        self.lo, self.hi = lo, hi
        if length is None:
            self.scale = 1.0
        else:
            fl = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_flops.json")))[f"c{cfg}"]
            self.scale = fl["full"] / fl["x".join(map(str, self.shape))]     # sample shifts per full-size shift
        self.cores = len(os.sched_getaffinity(0))
        from multiprocessing import get_context
        self.pool = get_context("fork").Pool(self.cores, initializer=_oracle_worker_init)

    def step(self, i0: int = 0):
        """One shift per core, all in parallel; returns (wall s, per-shift seconds)."""
        from kepgen import uniform_shifts
        sig = uniform_shifts(self.lo, self.hi, self.cores + 1)[:self.cores]
        sig = np.roll(sig, i0)
        t = time.time()
        res = self.pool.map(_oracle_worker, sig, chunksize=1)
        return time.time() - t, [r[0] for r in res]

    def describe(self):
        if self.scale == 1.0:
            return (f"c4 at full size (n={self.n}), one shift per core on {self.cores} cores in parallel, 1 BLAS "
                    f"thread each; measured, not scaled")
        return (f"c4 recipe on a {'x'.join(map(str, self.shape))} periodic sub-wire (n={self.n}), one shift per "
                f"core on {self.cores} cores in parallel, 1 BLAS thread each; wall time scaled to full-size "
                f"c4 shifts by the oracle's own flop ratio x{self.scale:.2f} (tests/golden/oracle_flops.json)")

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args, rank, world):
    """--impl reference: the oracle timed as it stands, on this run's config (rank 0 only)."""
    if rank != 0:
        return 0
    K, W = args.steps, args.warmup
    smp = OracleSample(args.config, args.ref_length)
    walls, per = [], []
    for i in range(W + K):
        wall, ts = smp.step(i)
        if i >= W:
            walls.append(wall)
            per += ts
    smp.close()
    wall = float(np.mean(walls))
    shift_eq = smp.cores / smp.scale                  # full-size c4 shift equivalents per step
    val = shift_eq / wall
    cfgd = workload_config(args.config, None, args.gpus, args.shifts_per_gpu)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "shifts/s", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": wall * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
            "cpu_baseline": {"value": val, "unit": "shifts/s", "cores": smp.cores, "kind": "oracle",
                             "sample": smp.describe(),
                             "sample_shifts_per_step": smp.cores,
                             "full_shift_equivalents_per_step": shift_eq,
                             "sample_seconds_per_shift_mean": float(np.mean(per)),
                             "extrapolated_seconds_per_full_shift_1core": float(np.mean(per)) * smp.scale},
            "e2e": {"value": val, "unit": "shifts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(cfg, length, pencil=None, bounds=None):
    smp = OracleSample(cfg, length, pencil, bounds)
    wall, ts = smp.step(0)
    smp.close()
    v = smp.cores / smp.scale / wall
    return {"value": v, "unit": "shifts/s", "cores": smp.cores, "kind": "oracle", "sample": smp.describe(),
            "sample_wall_s": wall, "sample_seconds_per_shift_mean": float(np.mean(ts)),
            "extrapolated_seconds_per_full_shift_1core": float(np.mean(ts)) * smp.scale}


# ----------------------------------------------------------------------------- multi-rank launch
def _relaunch_torchrun(n):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kep", choices=["kep", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--shifts-per-gpu", type=int, default=16)
    ap.add_argument("--shape", default=None, help="override lattice, e.g. 10x10x400 (development only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bracket", action="store_true", help="skip the time_to_bracket leg (ncu launch lists)")
    ap.add_argument("--cpu-length", type=int, default=150, help="sub-wire length of the cpu_baseline sample")
    ap.add_argument("--ref-length", type=int, default=100, help="sub-wire length of the reference-arm sample")
    ap.add_argument("--cpu-full", action="store_true",
                    help="cpu_baseline on the full-size c4 pencil (C shifts in parallel, ~15 min of host time)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return _relaunch_torchrun(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import kepgen
    from paper_1710_05134_b200 import Kep
    from paper_1710_05134_b200.multisection import Bracket, Multisection

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # NCCL init log (transport, NVLS) on stderr
        dist.init_process_group("nccl", device_id=dev)

    def log(*a):
        if rank == 0:
            print(*a, file=sys.stderr, flush=True)

    # ---- synthetic input: generated on rank 0, broadcast (replicated pencil; the path shards by shift)
    t0 = time.time()
    shape = tuple(int(x) for x in args.shape.split("x")) if args.shape else None
    meta = [None]
    if rank == 0:
        p = kepgen.config(args.config, shape=shape)
        lo, hi = kepgen.spectral_bounds(p)
        meta = [dict(n=p.n, nnz=p.nnz, k=p.k if p.k else int(0.3 * p.n), lo=lo, hi=hi, name=p.name)]
    if world > 1:
        dist.broadcast_object_list(meta, src=0)
    meta = meta[0]
    n, nnz = meta["n"], meta["nnz"]
    if rank == 0:
        colptr, rowidx, a, b = p.colptr, p.rowidx, p.a, p.b
    if world > 1:
        if rank == 0:
            tc = torch.from_numpy(colptr).to(dev); tr = torch.from_numpy(rowidx).to(dev)
            ta = torch.from_numpy(a).to(dev); tb = torch.from_numpy(b).to(dev)
        else:
            tc = torch.empty(n + 1, dtype=torch.int64, device=dev); tr = torch.empty(nnz, dtype=torch.int32, device=dev)
            ta = torch.empty(nnz, dtype=torch.float64, device=dev); tb = torch.empty(nnz, dtype=torch.float64, device=dev)
        for t in (tc, tr, ta, tb):
            dist.broadcast(t, src=0)
        colptr, rowidx, a, b = (t.cpu().numpy() for t in (tc, tr, ta, tb))
        del tc, tr, ta, tb
    t_gen = time.time() - t0
    log(f"[bench] input {meta['name']} n={n} nnz_lower={nnz} ready in {t_gen:.1f}s world={world}")

    S = args.shifts_per_gpu
    t0 = time.time()
    k = Kep(n, colptr, rowidx, max_batch=S, device=local_rank, profile=True)
    t_an = time.time() - t0
    ana = k.analysis()
    k.set_values(a, b)
    log(f"[bench] analysis {t_an:.1f}s: fronts={ana['n_fronts']} levels={ana['n_levels']} max_front={ana['max_front']} "
        f"flops/shift={ana['flops']:.3e} arena/shift={ana['arena_bytes']/1e9:.2f}GB batch={ana['batch']}")
    peak = fp64_peak_tflops() if rank == 0 else 0.0

    P = world * S
    initial = Bracket(meta["lo"], meta["hi"], 0, n)
    stats = dict(redo=0, delayed=0, evals=0, restarts=0, rounds=0)

    def nu_many(sig):
        nus, st, infos = k.inertia_many(sig, with_info=True)
        stats["redo"] += sum(i.n_redo for i in infos)
        stats["delayed"] += sum(i.n_delayed for i in infos)
        stats["evals"] += len(infos)
        return nus, st

    ms = Multisection(nu_many, k=meta["k"], shifts_per_rank=S, m_max=M_MAX, rank=rank, world=world,
                      device=dev if world > 1 else None)
    state = {"b": initial}

    def one_round(set_vals=None):
        if set_vals is not None:
            set_vals()
        state["b"], restarted = ms.step(state["b"], initial)
        stats["rounds"] += 1
        stats["restarts"] += int(restarted)

    for _ in range(args.warmup):
        one_round()
    torch.cuda.synchronize()
    k.reset_profile()
    stop = threading.Event()
    clocks = []
    th = threading.Thread(target=_clock_sampler, args=(stop, clocks, local_rank), daemon=True)
    th.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    w0 = time.time()
    for _ in range(args.steps):
        one_round()
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.time() - w0
    stop.set()
    dev_s = ev0.elapsed_time(ev1) / 1e3
    prof = k.profile()
    t_max = torch.tensor([dev_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_max = float(t_max.item())
    shifts_total = P * args.steps
    value = shifts_total / t_max

    # ---- e2e: host buffers through the C ABI, values re-uploaded from pinned memory every step
    e2e = None
    if not args.no_e2e:
        pa = torch.empty(nnz, dtype=torch.float64).pin_memory().numpy()
        pb = torch.empty(nnz, dtype=torch.float64).pin_memory().numpy()
        pa[:] = a
        pb[:] = b
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            one_round(set_vals=lambda: k.set_values(pa, pb))
        e1.record()
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": shifts_total / float(te.item()), "unit": "shifts/s",
               "h2d_bytes_per_step": int(2 * nnz * 8 + S * 8), "d2h_bytes_per_step": int(S * 8)}

    # ---- time to bracket: one complete stage 2 from the initial interval
    to_bracket = None
    if not args.no_bracket:
      if world > 1:
        dist.barrier()
      torch.cuda.synchronize()
      b2b0, b2b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
      b2b0.record()
      ms.trace.clear()
      fin = ms.run(initial)
      b2b1.record()
      torch.cuda.synchronize()
      tb = torch.tensor([b2b0.elapsed_time(b2b1) / 1e3], dtype=torch.float64, device=dev)
      if world > 1:
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
      to_bracket = {"seconds": float(tb.item()), "rounds": len(ms.trace), "shifts_per_round": P,
                  "k": meta["k"], "bracket": [fin.lo, fin.hi, fin.nu_lo, fin.nu_hi],
                  "table5_analogue": [{"interval": list(r.bracket[:2]), "index_range": list(r.bracket[2:]),
                                       "m": r.bracket[3] - r.bracket[2]} for r in ms.trace]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == 4 and not args.shape:
        if args.cpu_full:
            del k                                      # free device memory is irrelevant; host RAM is not
            cpu = cpu_baseline_leg(args.config, None, p, (meta["lo"], meta["hi"]))
        else:
            cpu = cpu_baseline_leg(args.config, args.cpu_length)

    if rank == 0:
        msd = prof["ms"]
        dom = max(msd, key=lambda x: msd[x])
        sch_t = (msd["schur"] + msd["schur_tma"]) / 1e3
        tma_t = msd["schur_tma"] / 1e3
        roof = {"bound": "tensor", "kernel": "k_schur + k_schur_tma + k_schur_small (a4, DMMA f64, every level)",
                "achieved": (prof["schur_flops"] / sch_t / 1e12) if sch_t > 0 else None,
                "peak": peak, "unit": "TFLOP/s",
                "frac": (prof["schur_flops"] / sch_t / 1e12 / peak) if sch_t > 0 and peak > 0 else None,
                "traffic": None,
                "traffic_note": "not measured by this run; ncu DRAM bytes of the Schur launches are in profiles/",
                "peak_source": "cuBLAS DGEMM 8192^3 measured live in bench.py (MEASURED_PEAKS.json has no FP64 entry)",
                "long_k_levels": {"kernel": "k_schur_tma (TMA-fed, levels averaging >= 128 pivots)",
                                  "achieved": (prof["schur_tma_flops"] / tma_t / 1e12) if tma_t > 0 else None,
                                  "frac": (prof["schur_tma_flops"] / tma_t / 1e12 / peak) if tma_t > 0 and peak > 0 else None,
                                  "share_of_schur_flops": prof["schur_tma_flops"] / max(prof["schur_flops"], 1.0)},
                "kernel_ms": msd, "kernel_launches": prof["launches"], "dominant_by_time": dom,
                "kernel_ms_note": "CUDA-event intervals per kernel class on the launching stream; on levels whose FS-size "
                                  "groups run on forked streams the 'fs' interval spans the whole k_fsp/k_fsu/k_l21 "
                                  "fork-join region (KEP_FS_STREAMS=0 separates the classes: profiles/r2_levels_c4.txt)",
                "schur_flops_alg": prof["schur_flops"]}
        launches = int(sum(prof["launches"].values()) + prof["other_launches"])
        fac_tflops = ana["flops"] * shifts_total / t_max / world / 1e12
        line = {"metric": METRIC, "value": value, "unit": "shifts/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(args.config, shape, world, S),
                "stats": {"nnz_lower": nnz, "flops_per_shift_alg": ana["flops"],
                          "factor_tflops_per_gpu": fac_tflops,
                          "factor_tflops_frac_of_fp64_peak": fac_tflops / peak if peak else None,
                          "fronts": ana["n_fronts"], "levels": ana["n_levels"], "max_front": ana["max_front"],
                          "arena_gb_per_shift": ana["arena_bytes"] / 1e9, "batch": ana["batch"],
                          "multisection_rounds": stats["rounds"], "restarts": stats["restarts"],
                          "delayed_pivots_per_shift": stats["delayed"] / max(stats["evals"], 1),
                          "fast_path_reruns_per_shift": stats["redo"] / max(stats["evals"], 1)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "time_to_bracket": to_bracket,
                "gpu_launches": launches, "clocks": _clock_summary(clocks), "wall_s": wall,
                "setup_s": {"generate": t_gen, "analyze": t_an}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

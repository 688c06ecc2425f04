"""bench.py — inertia evaluations nu_sigma/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kep|reference] [--config 4]

Workload (BASELINE.json configs[3], "c4"): the n = 1,500,000 quasi-1D
tight-binding pencil (10 x 10 x 3750 atoms, 4 orbitals, periodic z, cutoff
1.8), synthetic and seeded (kepgen).  One STEP is
one multisection round of stage 2 (Alg. 1' generalised to P = N x S shifts per
round): every rank factorises S = 16 shifts of the current
bracket (one LDL^T of A - sigma B each, rows a1-a5 of SURVEY.md §8), the int64
counts are all-gathered over NCCL and every rank applies the same bracket
update; a converged bracket (nu_u - nu_l <= m_max = 20) restarts from the
initial one.  Weak scaling: S shifts per GPU per step.

value = shifts factorised by all ranks / max-over-ranks device time of the K
timed steps (CUDA events on the library's stream, barrier + synchronize on
both sides).  e2e = the same through the public C-ABI call with HOST buffers:
every step uploads A and B values from pinned host memory (kep_set_values)
and reads the counts back.  The fronts (tens of GB) are far larger than L2,
so no L2 flush is needed between steps.
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
    """cuBLAS DGEMM 8192^3 best of 5 (the FP64 roofline denominator, measured live)."""
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


def traffic_per_launch(path=os.path.join(ROOT, "profiles", "r1_schur_traffic.json")):
    """DRAM bytes (read + write) per k_schur launch, from the committed ncu capture of this
    bench command (scripts/ncu_traffic.py); None if absent."""
    try:
        with open(path) as fh:
            return json.load(fh)["dram_bytes_per_launch"]
    except Exception:
        return None


# ----------------------------------------------------------------------------- CPU oracle leg
def cpu_oracle_sample(cfg: int, seconds_hint: float = 20.0):
    """Time the oracle (O-sparse, as it stands) on a bounded sample of the workload.

    Sample: the c4 recipe on a 10 x 10 x 150 sub-wire (n = 60,000), one shift,
    1 BLAS thread; scaled to full-size shifts/s by the oracle's own algorithmic
    flop count (full c4 / sample).  Returns (shifts_per_s_full, dict)."""
    import kepgen
    import oracle
    from oracle.sparse_mf import SparseOracle
    try:
        from threadpoolctl import threadpool_limits
    except Exception:                                  # pragma: no cover
        threadpool_limits = None
    base = dict(kepgen.CONFIGS[cfg])
    full_shape = base["shape"]
    sample_shape = (full_shape[0], full_shape[1], 150) if cfg == 4 else tuple(max(4, s // 3) for s in full_shape)
    base["shape"] = sample_shape
    p = kepgen.tb_pencil(**base)
    so = SparseOracle(p)
    lo, hi = kepgen.spectral_bounds(p)
    sig = 0.5 * (lo + hi)

    def flops_of(orc):
        piv, fs = orc.front_sizes()
        tot = 0.0
        for pp, ff in zip(piv, fs):
            c = ff - pp
            m = np.arange(c, ff, dtype=np.float64)
            tot += float(np.sum(m * m + 2 * m))
        return tot

    f_sample = flops_of(so)
    t0 = time.time()
    if threadpool_limits is not None:
        with threadpool_limits(1):
            r = so.inertia(sig)
    else:
        r = so.inertia(sig)
    dt = time.time() - t0
    # full-size oracle flops: the wire is uniform along z, so the oracle's
    # symbolic on the full pattern is replaced by the exact length ratio only
    # when the full symbolic would be too slow; here we compute it.
    pf = kepgen.tb_pencil(**dict(kepgen.CONFIGS[cfg])) if cfg != 4 else None
    if pf is not None:
        f_full = flops_of(SparseOracle(pf))
    else:
        f_full = f_sample * (full_shape[2] / sample_shape[2])
    scale = f_full / f_sample
    return 1.0 / (dt * scale), dict(sample=f"c{cfg} recipe on a {'x'.join(map(str, sample_shape))} lattice "
                                          f"(n={p.n}), 1 shift, 1 BLAS thread, scaled x{scale:.2f} by oracle flops",
                                   seconds=dt, nu=int(r.n_neg), oracle_flops_sample=f_sample, scale=scale)


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    K, W = args.steps, args.warmup
    times = []
    info = None
    for i in range(W + K):
        v, info = cpu_oracle_sample(args.config)
        if i >= W:
            times.append(1.0 / v)
    t = float(np.mean(times))
    val = 1.0 / t
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "shifts/s", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c{args.config}", "shifts_per_step": 1},
            "cpu_baseline": {"value": val, "unit": "shifts/s", "cores": 1, "kind": "oracle", "sample": info["sample"]},
            "e2e": {"value": val, "unit": "shifts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


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
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import kepgen
    from paper_1710_05134_b200 import Kep

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def log(*a):
        if rank == 0:
            print(*a, file=sys.stderr, flush=True)

    # ---- synthetic input: generated on rank 0, broadcast (replicated pencil, PAPER path shards by shift)
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
        dev = torch.device("cuda", local_rank)
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
    log(f"[bench] input {meta['name']} n={n} nnz_lower={nnz} ready in {t_gen:.1f}s")

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
    kk = meta["k"]
    lo0, hi0 = meta["lo"], meta["hi"]
    state = dict(lo=lo0, hi=hi0, nlo=0, nhi=n, rounds=0, restarts=0, redo=0, delayed=0, evals=0)

    def one_round(set_vals=None):
        """One multisection round: P interior shifts of [lo, hi), this rank takes i = rank mod world."""
        if set_vals is not None:
            set_vals()
        lo, hi = state["lo"], state["hi"]
        sig_all = lo + (np.arange(P) + 1.0) * (hi - lo) / (P + 1)
        mine = sig_all[rank::world]
        nus, st, infos = k.inertia_many(mine, with_info=True)
        state["redo"] += sum(i.n_redo for i in infos)
        state["delayed"] += sum(i.n_delayed for i in infos)
        state["evals"] += len(infos)
        nus = np.where(st == 0, nus, -1).astype(np.int64)
        if world > 1:
            t = torch.from_numpy(nus).cuda()
            out = torch.empty(world * len(nus), dtype=torch.int64, device=t.device)
            dist.all_gather_into_tensor(out, t)
            allv = out.cpu().numpy().reshape(world, -1).T.reshape(-1)      # back to shift order
        else:
            allv = nus
        # bracket update (SURVEY.md §8(c) reading 12): first pair with nu_a < k <= nu_b
        nus_full = np.concatenate([[state["nlo"]], allv, [state["nhi"]]])
        sig_full = np.concatenate([[lo], sig_all, [hi]])
        ok = np.all(allv >= 0)
        if ok:
            for j in range(len(sig_full) - 1):
                if nus_full[j] < kk <= nus_full[j + 1]:
                    state.update(lo=sig_full[j], hi=sig_full[j + 1], nlo=int(nus_full[j]), nhi=int(nus_full[j + 1]))
                    break
        state["rounds"] += 1
        if state["nhi"] - state["nlo"] <= M_MAX or not ok:
            state.update(lo=lo0, hi=hi0, nlo=0, nhi=n)
            state["restarts"] += 1

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
    t_max = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
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
        te = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": shifts_total / float(te.item()), "unit": "shifts/s",
               "h2d_bytes_per_step": int(2 * nnz * 8 + S * 8), "d2h_bytes_per_step": int(S * 8)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_oracle_sample(args.config)
        cpu = {"value": v, "unit": "shifts/s", "cores": 1, "kind": "oracle", "sample": info["sample"]}

    if rank == 0:
        ms = prof["ms"]
        dom = max(ms, key=lambda x: ms[x])
        sch_t = ms["schur"] / 1e3
        roof = {"bound": "tensor", "kernel": "k_schur (a4, DMMA f64)",
                "achieved": (prof["schur_flops"] / sch_t / 1e12) if sch_t > 0 else None,
                "peak": peak, "unit": "TFLOP/s",
                "frac": (prof["schur_flops"] / sch_t / 1e12 / peak) if sch_t > 0 and peak > 0 else None,
                "traffic": traffic_per_launch(),
                "peak_source": "cuBLAS DGEMM 8192^3 measured live in bench.py (MEASURED_PEAKS.json has no FP64 entry)",
                "kernel_ms": ms, "kernel_launches": prof["launches"], "dominant_by_time": dom,
                "schur_flops_alg": prof["schur_flops"]}
        launches = int(sum(prof["launches"].values()) + prof["other_launches"])
        fac_tflops = ana["flops"] * shifts_total / t_max / world / 1e12
        line = {"metric": METRIC, "value": value, "unit": "shifts/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"c{args.config}" + (f"-{args.shape}" if args.shape else ""), "n": n,
                           "nnz_lower": nnz, "shifts_per_gpu_per_step": S, "shifts_per_step": P,
                           "l2": "inputs larger than L2 (fronts ~GBs); no flush",
                           "flops_per_shift_alg": ana["flops"], "factor_tflops_per_gpu": fac_tflops,
                           "factor_tflops_frac_of_fp64_peak": fac_tflops / peak if peak else None,
                           "fronts": ana["n_fronts"], "levels": ana["n_levels"], "max_front": ana["max_front"],
                           "multisection_rounds": state["rounds"], "restarts": state["restarts"],
                           "delayed_pivots_per_shift": state["delayed"] / max(state["evals"], 1),
                           "fast_path_reruns_per_shift": state["redo"] / max(state["evals"], 1)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": _clock_summary(clocks), "wall_s": wall,
                "setup_s": {"generate": t_gen, "analyze": t_an}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Timings of the BASELINE.json configs beyond the bench's headline (C2).

    python tools/bench_configs.py [c1] [c3] [c4] [c5] [--cpu]

C1  mask SMC, 64^3 phantom pair, 500 particles x 20 iterations (the SPEC
    acceptance case); GPU register_smc e2e vs the CPU reference algorithm
    (oracle/smc.py + the bit-exact C kernel) on all host threads, same seed.
C3  register_sequence, mask mode, 30-frame 176x176x208 echo cycle,
    2000 particles x 50 iterations, then warp + score of all 30 frames.
C4  exhaustive search, default GridSpec (9^6 = 531,441 nodes), C2 pair.
C5  particle sweep 1k..256k on a 256^3 z-scored u8 pair: one measurement
    launch per P (evals/s, sampled/s, roofline fraction).
Writes one JSON object per config to stdout (and profiles/ via tee).
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def sync():
    torch.cuda.synchronize()


def truth_err(est, truth):
    d = est.to_array() - truth.to_array()
    return {"rot_err_deg": [round(math.degrees(x), 4) for x in d[:3]],
            "trans_err_mm": [round(float(x), 4) for x in d[3:]]}


def c1(cpu=False):
    from paper_2504_19930_b200 import (Executor, PhantomSpec, RigidParams, SmcConfig,
                                       make_pair, make_phantom, register_smc)

    seq, masks = make_phantom(PhantomSpec(dims=(64, 64, 64), frames=1, seed=0))
    truth = RigidParams(math.radians(5), math.radians(-8), math.radians(4), 6.0, -4.0, 3.0)
    case = make_pair(seq, masks, truth)
    tm, sm = case.target_masks[0], case.source_masks[0]
    cfg = SmcConfig(mode="mask", n_particles=500, n_iterations=20, seed=0)
    register_smc(tm, sm, cfg, Executor())  # warm-up
    times = []
    for _ in range(5):
        import copy

        a, b = copy.copy(tm), copy.copy(sm)
        for v in (a, b):
            if hasattr(v, "_er_device_cache"):
                object.__delattr__(v, "_er_device_cache")
        sync()
        t0 = time.perf_counter()
        est, tr = register_smc(a, b, cfg, Executor())
        sync()
        times.append(time.perf_counter() - t0)
    out = {"config": "C1 mask SMC 64^3, 500 x 20", "gpu_registration_ms": 1e3 * min(times),
           "gpu_registration_ms_median": 1e3 * sorted(times)[2],
           "evals_per_s": 500 * 64 ** 3 * 20 / min(times), **truth_err(est, truth)}
    if cpu:
        from oracle import kernels as ok
        from oracle import smc as osmc

        ok.build()
        geom = (tm.dims, tm.spacing, tm.origin)
        t0 = time.perf_counter()
        oest, _ = osmc.register(tm.data, sm.data, geom, geom,
                                osmc.Cfg(mode="mask", n_particles=500, n_iterations=20, seed=0))
        cpu_s = time.perf_counter() - t0
        d = est.to_array() - oest
        out.update({"cpu_reference_registration_s": cpu_s, "cpu_threads": ok.max_threads(),
                    "speedup_vs_cpu": cpu_s / min(times),
                    "gpu_vs_cpu_estimate_max_abs_diff": float(np.abs(d).max())})
    return out


def c3():
    from paper_2504_19930_b200 import Executor, SmcConfig, register_sequence
    from paper_2504_19930_b200.phantom_device import echo_case_device

    echo_case_device((40, 36, 44), frames=2)  # CUDA context + module load, not the generator
    sync()
    t0 = time.perf_counter()
    case = echo_case_device(frames=30, seed=0)
    sync()
    gen_s = time.perf_counter() - t0
    cfg = SmcConfig(mode="mask", n_particles=2000, n_iterations=50, seed=0)
    # warm-up on a 2-frame slice
    from paper_2504_19930_b200 import Sequence4

    register_sequence(Sequence4(case.target.frames[:2]), Sequence4(case.source.frames[:2]),
                      case.target_masks[:2], case.source_masks[:2],
                      SmcConfig(mode="mask", n_particles=64, n_iterations=2), Executor())
    # stage times: the calls register_sequence makes, on
    # a copy of the case with fresh raw arrays (so nothing is cached yet)
    from paper_2504_19930_b200 import Volume3, binarize, register_smc, to_matrix
    from paper_2504_19930_b200.pipeline import _normalize_frames, score_frames

    def fresh(vols):
        return [Volume3.from_u8(v.codec.raw.copy(), v.spacing, v.origin) for v in vols]

    # each stage: min over 3 repetitions, each on its own fresh copies (the
    # single-shot times vary with host-side allocator / GC state)
    samples = {"normalize_60_frames_s": [], "smc_s": [], "warp_and_score_30_frames_s": []}
    for r in range(3):
        ft, fs = Sequence4(fresh(case.target.frames)), Sequence4(fresh(case.source.frames))
        ftm, fsm = fresh(case.target_masks), fresh(case.source_masks)
        sync()
        t0 = time.perf_counter()
        nt, ns = _normalize_frames(ft), _normalize_frames(fs)
        sync()
        samples["normalize_60_frames_s"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        reg_t, reg_s = binarize(ftm[0], 0.5), binarize(fsm[0], 0.5)
        est, _ = register_smc(reg_t, reg_s, cfg, Executor(), trace_masks=(reg_t, reg_s))
        sync()
        samples["smc_s"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        score_frames(nt, ns, ftm, fsm, to_matrix(est, reg_t.physical_center()))
        sync()
        samples["warp_and_score_30_frames_s"].append(time.perf_counter() - t0)
    stages = {k: min(v) for k, v in samples.items()}
    stages["samples"] = samples
    walls = []
    for r in range(2):
        sync()
        t0 = time.perf_counter()
        rep = register_sequence(case.target, case.source, case.target_masks,
                                case.source_masks, cfg, Executor())
        sync()
        walls.append(time.perf_counter() - t0)
    return {"config": "C3 mask SMC + 30-frame 4D warp/score, 176x176x208, 2000 x 50",
            "register_sequence_s": min(walls), "register_sequence_samples_s": walls, "stages": stages, "phantom_generation_s": gen_s,
            "dsc_before_mean": rep.aggregates["dsc_before_mean"],
            "dsc_after_mean": rep.aggregates["dsc_after_mean"],
            "ncc_after_mean": rep.aggregates["ncc_after_mean"],
            "estimate_deg_mm": rep.estimate_deg_mm}


def c4():
    import bench
    from paper_2504_19930_b200 import Executor, GridSpec, register_exhaustive

    t, s, case = bench.make_workload()
    g = GridSpec()
    small = GridSpec(half_counts=(1, 1, 1, 1, 1, 1))
    register_exhaustive(t, s, small, Executor())
    sync()
    t0 = time.perf_counter()
    best, val = register_exhaustive(t, s, g, Executor())
    sync()
    wall = time.perf_counter() - t0
    return {"config": "C4 exhaustive 9^6 grid, C2 pair", "nodes": g.n_nodes,
            "seconds": wall, "evals_per_s": g.n_nodes * t.data.size / wall,
            "best_deg_mm": [math.degrees(x) for x in best.to_array()[:3]]
            + list(best.to_array()[3:]), "best_ncc": float(val)}


def c5(pmax=262144):
    from paper_2504_19930_b200 import SmcConfig, normalize_zscore
    from paper_2504_19930_b200 import smc as dsmc
    from paper_2504_19930_b200.backend import Executor
    from paper_2504_19930_b200.phantom_device import echo_case_device

    case = echo_case_device(dims=(256, 256, 256), spacing=(0.8, 0.8, 0.8), frames=1, seed=0)
    t = normalize_zscore(case.target.frames[0])
    s = normalize_zscore(case.source.frames[0])
    rows = []
    p = 1024
    while p <= pmax:
        cfg = SmcConfig(mode="image", n_particles=p, n_iterations=1, seed=0)
        run = dsmc.DeviceSmcRun(t, s, cfg, Executor())
        run.predict(0)
        run.measure()
        sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run.measure()
        e1.record()
        sync()
        ms = e0.elapsed_time(e1)
        nin = float(run.n_local[:p].sum().item())
        rows.append({"particles": p, "ms": ms, "evals_per_s": p * t.data.size / (ms * 1e-3),
                     "sampled_per_s": nin / (ms * 1e-3),
                     "hbm_frac_9B": nin * 9 / (ms * 1e-3) / 6535.4e9})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        del run
        torch.cuda.empty_cache()
        p *= 4
    return {"config": "C5 particle sweep on 256^3, 1 GPU", "rows": rows}


def scaling(p_list=(2000, 65536), n_list=(1, 2, 4, 8), reps=5):
    """Per-rank work of an N-GPU run, measured on this GPU: each rank runs
    predict + update for all P particles (replicated) and affines + the
    measurement for its shard of ceil(P/N) particles.  The NCCL all-gather of
    P doubles is NOT measured here (one GPU); it is added as an explicit
    estimate from the measured NVLink peer bandwidth in B200_PROFILING.md
    (770 GB/s per direction) plus 20 us of launch latency.  A projection, not
    a multi-GPU measurement."""
    import bench
    from paper_2504_19930_b200 import SmcConfig
    from paper_2504_19930_b200 import dist, smc as dsmc
    from paper_2504_19930_b200.backend import Executor

    t, s, _ = bench.make_workload()
    nvox = t.data.size
    out = []

    def local_gather(local, out):  # the NCCL exchange's cost is estimated below
        out[: local.numel()].copy_(local)
        return out

    dsmc.dist.allgather_packed = local_gather
    for P in p_list:
        cfg = SmcConfig(mode="image", n_particles=P, n_iterations=reps + 2, seed=0)
        base = None
        for N in n_list:
            run = dsmc.DeviceSmcRun(t, s, cfg, Executor())
            run.plan = dist.ShardPlan(P, N, 0)  # rank 0 holds the first (largest) shard
            # rank 0's packed block [z | flags] and the gathered buffer of N blocks
            S = run.plan.shard
            run.block = dist.packed_block_bytes(S)
            run.zd_local = torch.zeros(run.block, dtype=torch.uint8, device=run.dev)
            run.z_local = run.zd_local[: 8 * S].view(torch.float64)
            run.dg_local = run.zd_local[8 * S: 9 * S]
            run.zd_all = torch.zeros(run.block * N, dtype=torch.uint8, device=run.dev)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            for k in range(2):
                run.step(k)
            sync()
            ev[0].record()
            for k in range(2, 2 + reps):
                run.step(k)
            ev[1].record()
            sync()
            ms = ev[0].elapsed_time(ev[1]) / reps
            gather_ms = 0.0 if N == 1 else 0.020 + P * 8 * (N - 1) / N / 770e9 * 1e3
            it_ms = ms + gather_ms
            evals = P * nvox / (it_ms * 1e-3)
            if base is None:
                base = evals
            out.append({"particles": P, "gpus": N, "rank0_iteration_ms": round(ms, 3),
                        "allgather_ms_estimate": round(gather_ms, 4),
                        "projected_evals_per_s": evals, "projected_efficiency": evals / base / N})
            print(json.dumps(out[-1]), file=sys.stderr, flush=True)
            del run
            torch.cuda.empty_cache()
    return {"config": "scaling projection (per-rank work measured on one B200)", "rows": out}


if __name__ == "__main__":
    which = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c1", "c3", "c4", "c5"]
    for w in which:
        fn = globals()[w]
        res = fn(cpu=("--cpu" in sys.argv)) if w == "c1" else fn()
        print(json.dumps(res), flush=True)

#!/usr/bin/env python
"""bench.py -- candidate merge-error evaluations/s on B200 (arXiv 2601.11626).

Headline workload (N=1): BASELINE.json's largest single-GPU config, configs[3]
("config4"): N=64 fp32 blocks of 4096x4096 (16 synthetic layers x Q/K/V/O,
4 layer groups sharing rank-256 left subspaces), r = 256, TRUNC operand (A6);
all 2016 candidate pairs (base = the block of larger norm, A7) with all three
estimators (Weyl, residual, incremental).  SURVEY.md §8(d):
  * the unit is one (base, appended) evaluation producing the requested kinds;
  * one step = one cmsvd_pair_errors pass over all P pairs (device-resident
    pairs and outputs, S3-S9); value = P * K / (sum of the K steps' CUDA-event
    times on the library's stream), L2 flushed by a 256 MiB write before every
    step (outside the step's events; the step reads 0.5 GB of bases/operands);
  * the one-time S1 (register, energies) and S2 (block spectra) are timed
    separately (CUDA events) and reported under "one_time", not in the rate;
  * four per-kind rates: Weyl-only, residual-only, incremental-only, all three.
e2e = the same metric through the C ABI with HOST buffers: every step
register(pinned host blocks) + block_spectra + pair_errors(host pairs -> host
outputs), host wall clock (copies and the one-time work inside).
"extras": the config-2 line (all 8128 pairs) and greedy wall times.

Multi-GPU (torchrun): "replicas only": each rank evaluates its own
independent collection (seed offset by rank) -- no data-path collective; the
job time is the max over ranks (all_reduce of the timings only).

--impl reference runs the float64 CPU oracle (oracle/) on a bounded sample of
the same workload: the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import signal
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "candidate merge-error evaluations/sec at 1 B200; % of tensor/HBM roofline"
UNIT = "evals/s"
KIND_NAMES = {1: "weyl", 2: "residual", 4: "incremental", 7: "all"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cmsvd", choices=["cmsvd", "reference"])
    ap.add_argument("--config", default="config4")
    ap.add_argument("--kind-steps", type=int, default=3, help="timed steps per single-kind rate")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=256, help="pairs timed for the oracle cpu_baseline (configs 1/2/5)")
    ap.add_argument("--ref-sample", type=int, default=48, help="pairs per --impl reference step (configs 1/2/5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {}


# Own microbenchmarks of the SIMT pipes on this pool's B200 (tools/peaks.cu, profiles/peaks_r01.txt):
# FFMA 72.5 TF/s, DFMA 33.96 TF/s.  MEASURED_PEAKS.json has no FP64 / FP32-SIMT figure.
DFMA_TFLOPS = 33.96
FFMA_TFLOPS = 72.54


def tf32_fp32eq_tflops() -> float:
    """fp32-equivalent 3xTF32 tensor peak: MEASURED_PEAKS.json dense bf16 burst x the nominal TF32/BF16
    ratio (1.125/2.25 PF dense) / 3 MMAs per useful product; fallback 2250/2/3."""
    return load_peaks().get("bf16_tflops", 2250.0) * 0.5 / 3.0


def hbm_gbs() -> float:
    return load_peaks().get("hbm_gbs", 6650.0)


def workload(name: str, rank: int):
    if name == "config2":
        return synth.config2(seed=1 + 1000 * rank)
    if name == "config1":
        return synth.config1(seed=0 + 1000 * rank)
    if name.startswith("config5"):
        N = 2048 if "N2048" in name else 512
        r = 64 if name.endswith("r64") else 16
        return synth.config5(seed=4 + 1000 * rank, N=N, r=r)
    if name == "config3":
        return synth.config3(seed=2 + 1000 * rank)
    if name == "config4":
        return synth.config4(seed=3 + 1000 * rank)
    raise SystemExit(f"unknown config {name}")


def is_big(name: str) -> bool:
    """configs 3/4: square weight-like blocks, TRUNC operand (A6), A22 spectra."""
    return name in ("config3", "config4")


def norm_order(E):
    return np.array(sorted(range(len(E)), key=lambda i: (-E[i], i)))


def max_over_ranks(dist, x: float, dev=None) -> float:
    """Max of a host scalar over all ranks (timings: the job is as slow as its slowest rank)."""
    if not dist:
        return x
    import torch
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 0, 1, 0, None
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(local)
    dist.init_process_group(backend=backend)
    return rank, ws, local, dist


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.send_signal(signal.SIGTERM)
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [r for r in rows if r[2] > 200.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in load for k, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load)}


# ---------------------------------------------------------------------------
# Algorithmic work model: flops / bytes of all P pairs of one step
# ---------------------------------------------------------------------------
def work_model(col, pairs, blk_rank, big):
    m = float(col.m)
    rr_b = np.minimum(col.r, blk_rank).astype(np.float64)
    # projection basis of each base: the full numerical range (tall-thin) or U_r (A22 blocks);
    # appended operand width: the raw block (RAW) or its rank-r factor (TRUNC)
    q = (rr_b if big else blk_rank.astype(np.float64))[pairs[:, 0]]
    w = rr_b[pairs[:, 1]] if big else np.full(pairs.shape[0], float(col.n))
    nG = rr_b[pairs[:, 0]] + w
    flops = {
        "eig_G": float(np.sum(4.0 / 3.0 * nG ** 3)),       # Householder tridiagonalisation of the core Gram
        "eig_W": float(np.sum(4.0 / 3.0 * w ** 3)),
        "gram_W": float(np.sum(m * w * (w + 1))),
        "gram_ZZ": float(np.sum(q * w * (w + 1))),
        "proj_Z": float(np.sum(2.0 * m * q * w)),
        "resid_R": float(np.sum(2.0 * m * q * w)),
        "pair_tc": float(np.sum(4.0 * m * q * w + m * w * (w + 1))),   # Z, R', W' useful flops
    }
    # unique HBM bytes of the materialised residual R' = F - Q Z (read Q, Z, F; write R')
    nbytes = {"resid_R": float(np.sum(4.0 * (m * q + q * w + 2 * m * w)))}
    # two-stage reduction of the core Grams with n > 160 (k_sbr.cu): per panel t the trailing block has
    # n_p = n - 16 (t + 1) rows; the symmetric product streams the full n_p^2 block once, the rank-32 update
    # reads and writes its lower triangle (8 B per element)
    big_n = nG[nG > 160]
    if big_n.size:
        sym_b = syr_b = sym_f = syr_f = 0.0
        for nn in np.unique(big_n):
            cnt = float(np.sum(big_n == nn))
            npv = nn - 16.0 * np.arange(1, int((nn - 18) // 16) + 2)
            npv = npv[npv >= 2]
            sym_b += cnt * float(np.sum(8.0 * npv ** 2))
            syr_b += cnt * float(np.sum(16.0 * npv * (npv + 1) / 2))
            sym_f += cnt * float(np.sum(2.0 * 16 * npv ** 2))
            syr_f += cnt * float(np.sum(2.0 * 32 * npv * (npv + 1) / 2))
        nbytes["sbr_symm"], nbytes["sbr_syr2k"] = sym_b, syr_b
        flops["sbr_symm"], flops["sbr_syr2k"] = sym_f, syr_f
    return flops, nbytes


def categorize(prof, flops, nbytes, total_ms, steps, tiles):
    tc_peak = tf32_fp32eq_tflops()
    peaks = {"eig_G": DFMA_TFLOPS, "eig_W": DFMA_TFLOPS, "gram_W": tc_peak if tiles else DFMA_TFLOPS,
             "sbr_symm": DFMA_TFLOPS, "sbr_syr2k": DFMA_TFLOPS,
             "gram_ZZ": DFMA_TFLOPS, "proj_Z": tc_peak if tiles else FFMA_TFLOPS,
             "resid_R": tc_peak if tiles else FFMA_TFLOPS, "pair_tc": tc_peak}
    kernels = {}
    for name, (ms, cnt) in prof.items():
        if cnt == 0:
            continue
        e = {"ms_total": ms, "launches": cnt, "share": ms / max(total_ms, 1e-9)}
        if name in flops:
            # flops[name] covers all P pairs of one step; a step may launch a category several times
            # (pair-workspace chunks), so the rate is per step, not per launch group
            e["tflops"] = flops[name] * steps / (ms * 1e-3) / 1e12
            e["frac_of_peak"] = e["tflops"] / peaks[name]
            e["peak_tflops"] = peaks[name]
        if name in nbytes:
            e["gbs"] = nbytes[name] * steps / (ms * 1e-3) / 1e9
            e["frac_of_hbm"] = e["gbs"] / hbm_gbs()
        kernels[name] = e
    return kernels, peaks, tc_peak


def roofline_entry(name, e, peaks, tc_peak, traffic):
    tensor = peaks.get(name) == tc_peak
    return {"bound": "tensor" if tensor else "alu", "kernel": name, "achieved": e["tflops"],
            "peak": peaks[name], "unit": "TFLOP/s", "frac": e["frac_of_peak"], "traffic": traffic,
            "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                            "(profiles/ncu_traffic.json)",
            "peak_source": ("MEASURED_PEAKS.json bf16 burst x 0.5 (nominal TF32/BF16) / 3 (3xTF32 MMAs per useful "
                            "fp32 product)") if tensor else
                           ("own DFMA/FFMA microbenchmark (tools/peaks.cu, profiles/peaks_r01.txt); "
                            "MEASURED_PEAKS.json has no FP64 / FP32-SIMT peak"),
            "algorithmic": "Householder tridiagonalisation 4/3 n^3 flops per n x n core Gram (n = r' + w)"
            if name.startswith("eig") else "2 m q w (GEMM) / m w (w+1) (SYRK) flops per pair"}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the float64 oracle, bounded samples
# ---------------------------------------------------------------------------
def big_sample_ids(E, k):
    """Deterministic block subset of a config-3/4 collection: the k largest-norm blocks."""
    return [int(i) for i in norm_order(E)[:k]]


def cpu_baseline(col, pairs, r, sample, E, big=False):
    import oracle
    P = pairs.shape[0]
    if big:
        # configs 3/4: the oracle's exact m x m Gram eigendecompositions cost ~20 s per 4096^2 block, so
        # the sample is the ordered pairs among the 2 largest-norm blocks (the first pair of the list and
        # its reverse); their spectra are timed and reported per block, outside the rate (like S2)
        ids = big_sample_ids(E, 2)
        t0 = time.perf_counter()
        sp = oracle.block_spectra(np.ascontiguousarray(col.blocks[ids]), nvec=r)
        t_spec = time.perf_counter() - t0
        sub = np.array([[0, 1], [1, 0]], np.int32)
        S = sub.shape[0]
        t0 = time.perf_counter()
        oracle.pair_errors(sp, sub, r, 7, oracle.TRUNC)
        t_pairs = time.perf_counter() - t0
        what = (f"the {S} ordered pairs between the 2 largest-norm blocks {ids} (TRUNC operand, all 3 estimators, "
                f"float64 oracle, one pair per thread); their block spectra took {t_spec:.1f} s "
                f"({t_spec / len(ids):.1f} s per block, one-time, not in the rate)")
    else:
        t0 = time.perf_counter()
        sp = oracle.block_spectra(col.blocks)
        t_spec = time.perf_counter() - t0
        S = min(sample, P)
        t0 = time.perf_counter()
        oracle.pair_errors(sp, pairs[:S], r, 7, oracle.RAW)
        t_pairs = time.perf_counter() - t0
        what = (f"first {S} of the {P} norm-ordered pairs, all 3 estimators, float64 oracle (OpenMP over "
                f"pairs); its block spectra took {t_spec:.2f} s for all {col.N} blocks (one-time, not in the rate)")
    return {"value": S / t_pairs, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "sample": what,
            "seconds": t_pairs, "spectra_seconds": t_spec}


def run_reference(args):
    rank, ws, local, dist = dist_init()
    if rank != 0:
        return
    import oracle
    col = workload(args.config, 0)
    big = is_big(args.config)
    E = np.array([oracle.energy(col.blocks[i]) for i in range(col.N)])
    t0 = time.perf_counter()
    if big:
        # one-time S2 on a deterministic block subset (the 3 largest-norm blocks: 6 ordered pairs)
        ids = big_sample_ids(E, 3)
        sp = oracle.block_spectra(np.ascontiguousarray(col.blocks[ids]), nvec=col.r)
        pairs = np.array([[a, b] for a in range(3) for b in range(3) if a != b], np.int32)
        operand, S = oracle.TRUNC, pairs.shape[0]
        sample = (f"per step the {S} ordered pairs among the 3 largest-norm blocks {ids} (TRUNC, all 3 estimators, "
                  f"one pair per thread); their oracle spectra are one-time, outside the steps")
    else:
        sp = oracle.block_spectra(col.blocks)
        pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
        operand, S = oracle.RAW, min(args.ref_sample, pairs.shape[0])
        sample = (f"{S} pairs per step of the {pairs.shape[0]} norm-ordered pairs (all 3 estimators); "
                  f"the oracle block spectra are one-time, outside the steps")
    t_spec = time.perf_counter() - t0
    for w in range(args.warmup):
        oracle.pair_errors(sp, pairs[:1], col.r, 7, operand)
    t0 = time.perf_counter()
    for k in range(args.steps):
        off = (k * S) % pairs.shape[0]
        sub = pairs[off:off + S] if off + S <= pairs.shape[0] else np.concatenate([pairs[off:], pairs[:off + S - pairs.shape[0]]])
        oracle.pair_errors(sp, sub, col.r, 7, operand)
    dt = time.perf_counter() - t0
    value = S * args.steps / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": args.config, "N": col.N, "m": col.m, "n": col.n, "r": col.r,
                      "pairs_per_step": S, "kinds": "weyl+residual+incremental",
                      "operand": "TRUNC" if big else "RAW"},
           "one_time": {"oracle_spectra_s": t_spec},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def make_out(torch, P, r, dev):
    return {"err2": torch.empty((P, 3), dtype=torch.float64, device=dev),
            "total": torch.empty(P, dtype=torch.float64, device=dev),
            "sigma_tilde": torch.empty((P, r), dtype=torch.float32, device=dev),
            "mu": torch.empty((P, r), dtype=torch.float32, device=dev)}


def timed_steps(torch, stream, fn, steps, flush):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.zero_()
        ev[k][0].record(stream)
        fn()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def secondary_line(cm, torch, stream, dev, local, name, steps, flush):
    """Pair-pass rate of another config (all pairs, all three kinds), one-time S1/S2 beside it."""
    col = workload(name, 0)
    big = is_big(name)
    with cm.Context(local, stream.cuda_stream) as ctx:
        blocks_d = torch.from_numpy(col.blocks).to(dev)
        t0 = time.perf_counter()
        ctx.register(blocks_d)
        E, _, _ = ctx.block_spectra(col.r)
        torch.cuda.synchronize()
        t_once = time.perf_counter() - t0
        pairs = synth.all_pairs_by_norm_order(norm_order(E))
        P = pairs.shape[0]
        pairs_d = torch.from_numpy(pairs).to(dev)
        out = make_out(torch, P, col.r, dev)
        fn = lambda: ctx.pair_errors(pairs_d, out=out, operand=cm.TRUNC if big else cm.RAW)  # noqa: E731
        for _ in range(3):
            fn()
        times = timed_steps(torch, stream, fn, steps, flush)
    return {"workload": name, "pairs": P, "value": P * steps / (sum(times) / 1e3), "unit": UNIT,
            "ms_per_step": sum(times) / steps, "one_time_register_spectra_s": t_once}


def greedy_runs(cm, torch, stream, dev, local, runs):
    out = {}
    for name, alg, srt, eps, knn in runs:
        col = workload(name, 0)
        big = is_big(name)
        with cm.Context(local, stream.cuda_stream) as ctx:
            ctx.register(torch.from_numpy(col.blocks).to(dev))
            ctx.block_spectra(col.r)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = ctx.cluster(alg, eps, sort=srt, knn=knn, operand=cm.TRUNC if big else cm.RAW)
            ms = 1e3 * (time.perf_counter() - t0)
        out[f"{name}_alg{alg}_sort{srt}_knn{knn}_eps{eps}"] = {
            "ms": ms, "clusters": len(res["clusters"]), "n_evals": res["n_evals"],
            "ms_per_eval": ms / max(1, res["n_evals"])}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    rank, ws, local, dist = dist_init()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_2601_11626_b200 as cm
    # a dedicated (non-default) stream: the library enqueues on it and every CUDA event of the timed
    # region is recorded on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    col = workload(args.config, rank)
    r = col.r
    big = is_big(args.config)
    operand = cm.TRUNC if big else cm.RAW
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ctx = cm.Context(local, stream.cuda_stream)
    blocks_d = torch.from_numpy(col.blocks).to(dev)

    # ---- one-time S1 (register: copy into the arena + fp64 energies) and S2 (block spectra) ----
    ctx.register(blocks_d)
    ctx.block_spectra(r)
    torch.cuda.synchronize()
    ctx.profile(True)
    t_s1 = timed_steps(torch, stream, lambda: ctx.register(blocks_d), 1, flush)[0]
    prof_s1 = ctx.profile_read()
    ctx.profile(False)
    t_s2 = timed_steps(torch, stream, lambda: ctx.block_spectra(r), 1, flush)[0]
    E, _, blk_rank = ctx.block_spectra(r)
    s1_kernel_ms = prof_s1.get("energy", (0.0, 0))[0]
    one_time = {"s1_register_ms": t_s1, "s1_energy_kernel_ms": s1_kernel_ms,
                "s1_energy_gbs": col.blocks.nbytes / (s1_kernel_ms * 1e-3) / 1e9 if s1_kernel_ms else None,
                "s2_block_spectra_ms": t_s2,
                "note": "register = D2D copy into the library arena + energy kernel; not in the rate (§8(d))"}

    pairs = synth.all_pairs_by_norm_order(norm_order(E))
    P = pairs.shape[0]
    pairs_d = torch.from_numpy(pairs).to(dev)
    out = make_out(torch, P, r, dev)

    def step(kinds=cm.ALL):
        ctx.pair_errors(pairs_d, out=out, operand=operand, kinds=kinds)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    ctx.profile(True)
    with ClockSampler(local) as clk:
        times = timed_steps(torch, stream, step, args.steps, flush)
    prof = ctx.profile_read()
    ctx.profile(False)
    launches = ctx.launches - launches0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = max_over_ranks(dist, sum(times), dev)
    value = P * args.steps * ws / (total_ms / 1e3)

    # ---- per-kind rates (same pairs, kinds = one estimator) ----
    per_kind = {"all": value}
    for kinds in (cm.WEYL, cm.RESIDUAL, cm.INCREMENTAL):
        fn = lambda k=kinds: step(k)  # noqa: E731
        fn()
        tk = timed_steps(torch, stream, fn, args.kind_steps, flush)
        tk_ms = max_over_ranks(dist, sum(tk), dev)
        per_kind[KIND_NAMES[kinds]] = P * args.kind_steps * ws / (tk_ms / 1e3)

    # ---- roofline of the dominant kernel category (live CUDA events) + the other contractions ----
    flops, nbytes = work_model(col, pairs, blk_rank, big)
    tiles = big or col.n > 128 or r > 128
    kernels, peaks, tc_peak = categorize(prof, flops, nbytes, total_ms, args.steps, tiles)
    dom_all = max(kernels, key=lambda k: kernels[k]["ms_total"])
    dom = max((k for k in kernels if k in flops), key=lambda k: kernels[k]["ms_total"], default=dom_all)
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")   # dram bytes per launch from ncu --set full
    traffic = json.load(open(tfile)).get(args.config, {}) if os.path.exists(tfile) else {}
    roof = roofline_entry(dom, kernels[dom], peaks, tc_peak, traffic.get(dom)) if dom in flops else \
        {"bound": "alu", "kernel": dom, "achieved": None, "peak": None, "unit": "TFLOP/s", "frac": None,
         "traffic": None}
    others = [roofline_entry(k, kernels[k], peaks, tc_peak, traffic.get(k))
              for k in ("proj_Z", "resid_R", "gram_W", "pair_tc", "sbr_symm", "sbr_syr2k")
              if k in kernels and k in flops and k != dom]
    for o in others:
        if o["kernel"] in nbytes:
            e = kernels[o["kernel"]]
            o["hbm"] = {"achieved": e["gbs"], "peak": hbm_gbs(), "unit": "GB/s", "frac": e["frac_of_hbm"],
                        "algorithmic": "read Q, Z, F + write R' per pair (4 B each)" if o["kernel"] == "resid_R" else
                        "per panel: the n_p^2 trailing block read once (symm) / its lower triangle read + "
                        "written (syr2k), 8 B per element"}
    if one_time["s1_energy_gbs"]:
        others.append({"bound": "hbm", "kernel": "energy (S1, one-time)", "achieved": one_time["s1_energy_gbs"],
                       "peak": hbm_gbs(), "unit": "GB/s", "frac": one_time["s1_energy_gbs"] / hbm_gbs(),
                       "traffic": None, "algorithmic": "4 B read per fp32 element of the collection"})

    result = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
              "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
              "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
              "config": {"workload": args.config, "N": col.N, "m": col.m, "n": col.n, "r": r, "pairs": P,
                         "kinds": "weyl+residual+incremental", "operand": "TRUNC" if big else "RAW",
                         "step": "cmsvd_pair_errors over all pairs (S3-S9), device-resident pairs/outputs; "
                                 "one-time S1/S2 timed separately",
                         "l2": "flushed (256 MiB write) before every step, outside the step events",
                         "parallelism": f"replicas x{ws} (independent collections, no collective)"},
              "per_kind": per_kind, "one_time": one_time,
              "gpu_launches": launches, "roofline": roof, "rooflines_other": others, "kernels": kernels,
              "dominant_category": dom_all, "step_ms": times}
    result["clocks"] = clk.summary()

    # ---- e2e through the C ABI with host buffers ----
    if not args.no_e2e:
        pinned = torch.from_numpy(col.blocks).pin_memory()
        pairs_h = np.ascontiguousarray(pairs)
        ctx2 = cm.Context(local, stream.cuda_stream)
        ctx2.register(pinned)
        ctx2.block_spectra(r)
        ctx2.pair_errors(pairs_h, operand=operand)
        torch.cuda.synchronize()
        ks = max(1, args.e2e_steps)
        t0 = time.perf_counter()
        for _ in range(ks):
            ctx2.register(pinned)
            ctx2.block_spectra(r)
            res_h = ctx2.pair_errors(pairs_h, operand=operand)
        t_e2e = max_over_ranks(dist, time.perf_counter() - t0, dev)
        h2d = col.blocks.nbytes + pairs_h.nbytes
        d2h = res_h["err2"].nbytes + res_h["total"].nbytes + res_h["sigma_tilde"].nbytes + res_h["mu"].nbytes + \
            col.N * (8 + 4 * r + 4)
        result["e2e"] = {"value": P * ks * ws / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                         "d2h_bytes_per_step": int(d2h), "steps": ks,
                         "path": "per step: cmsvd_register(pinned host blocks) + cmsvd_block_spectra + "
                                 "cmsvd_pair_errors(host pairs -> host outputs), host wall clock"}
        ctx2.close()
    ctx.close()
    del blocks_d

    # ---- extras: the config-2 line and greedy wall times (rank 0) ----
    if not args.no_extras and rank == 0:
        ex = {}
        if args.config != "config2":
            ex["config2"] = secondary_line(cm, torch, stream, dev, local, "config2", args.steps, flush)
        runs = [("config2", cm.ALG_APPROX, cm.SORT_RESIDUAL, 0.05, 1),
                ("config2", cm.ALG_RESIDUAL, cm.SORT_FROBENIUS, 0.05, 1),
                ("config5_N2048_r16", cm.ALG_APPROX, cm.SORT_RESIDUAL, 0.1, 16)]
        if args.config == "config4":
            runs.append(("config4", cm.ALG_APPROX, cm.SORT_RESIDUAL, 0.15, 1))
        ex["greedy"] = greedy_runs(cm, torch, stream, dev, local, runs)
        result["extras"] = ex

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(col, pairs, r, args.cpu_sample, E, big=big)
    if rank == 0:
        print(json.dumps(result))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

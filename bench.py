#!/usr/bin/env python
"""bench.py -- candidate merge-error evaluations/s on B200 (arXiv 2601.11626).

Workload (N=1): BASELINE.json configs[1] ("config2"): N=128 fp32 blocks of
512x128, 8 hidden groups, r = 32; all 8128 candidate pairs (base = the block
of larger norm, A7) with all three estimators (Weyl, residual, incremental).
One step = one pass of the whole hot path over the collection:
  cmsvd_register (S1, device-resident input copied into the arena + fp64
  energies) -> cmsvd_block_spectra (S2) -> cmsvd_pair_errors (S3-S9) with
  device-resident pairs and outputs.
value = pair evaluations / device time (CUDA events on the library's stream,
L2 flushed by a 256 MiB write before every step, outside the step's events).

Multi-GPU (torchrun): weak scaling, each rank evaluates its own independent
collection (seed offset by rank) -- no data-path collective; the job time is
the max over ranks (gloo/nccl all_reduce of the timings only).

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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cmsvd", choices=["cmsvd", "reference"])
    ap.add_argument("--config", default="config2")
    ap.add_argument("--cpu-sample", type=int, default=256, help="pairs timed for the oracle cpu_baseline")
    ap.add_argument("--ref-sample", type=int, default=48, help="pairs per --impl reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-greedy", action="store_true")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {}
    if os.path.exists(p):
        peaks = json.load(open(p))
    return peaks


# Own microbenchmark of the SIMT pipes on this pool's B200 (tools/peaks.cu,
# profiles/peaks_r01.txt): FFMA 72.5 TF/s, DFMA 33.96 TF/s.
DFMA_TFLOPS = 33.96
FFMA_TFLOPS = 72.54


def tf32_fp32eq_tflops() -> float:
    """fp32-equivalent 3xTF32 tensor peak: MEASURED_PEAKS.json dense bf16 burst x the nominal TF32/BF16
    ratio (1.125/2.25 PF dense) / 3 MMAs per useful product; fallback 2250/2/3."""
    bf16 = load_peaks().get("bf16_tflops", 2250.0)
    return bf16 * 0.5 / 3.0


def workload(name: str, rank: int):
    if name == "config2":
        col = synth.config2(seed=1 + 1000 * rank)
    elif name == "config1":
        col = synth.config1(seed=0 + 1000 * rank)
    elif name.startswith("config5"):
        r = 64 if name.endswith("r64") else 16
        col = synth.config5(seed=4 + 1000 * rank, N=512, r=r)
    elif name == "config3":
        col = synth.config3(seed=2 + 1000 * rank)
    elif name == "config4":
        col = synth.config4(seed=3 + 1000 * rank)
    else:
        raise SystemExit(f"unknown config {name}")
    return col


def is_big(name: str) -> bool:
    """configs 3/4: square weight-like blocks, TRUNC operand (A6), A22 spectra."""
    return name in ("config3", "config4")


def max_over_ranks(dist, x: float, dev=None) -> float:
    """Max of a host scalar over all ranks (timings: the job is as slow as its slowest rank)."""
    if not dist:
        return x
    import torch
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_init(args):
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


def tridiag_flops(n):
    return 4.0 / 3.0 * n ** 3


def cpu_baseline(col, pairs, r, sample, timeout_s=40.0, big=False):
    import oracle
    P = pairs.shape[0]
    if big:
        # configs 3/4: the oracle's exact m x m Gram eigendecompositions cost seconds per block, so the
        # sample is the pairs among the first three norm-ordered blocks, their spectra scaled to all N
        ids = list(dict.fromkeys(int(b) for pr in pairs[:3] for b in pr))[:3]
        sub = np.array([[a, b] for a in range(len(ids)) for b in range(len(ids)) if a != b], np.int32)
        t0 = time.perf_counter()
        sp = oracle.block_spectra(np.ascontiguousarray(col.blocks[ids]))
        t_spec = (time.perf_counter() - t0) * col.N / len(ids)
        S = sub.shape[0]
        t0 = time.perf_counter()
        oracle.pair_errors(sp, sub, r, 7, oracle.TRUNC)
        t_pairs = time.perf_counter() - t0
        what = (f"the {S} ordered pairs among blocks {ids} (TRUNC operand, all 3 estimators, float64 oracle); "
                f"block spectra measured on those {len(ids)} blocks, scaled to all {col.N} ({t_spec:.1f} s) "
                f"and prorated by {S}/{P}")
    else:
        t0 = time.perf_counter()
        sp = oracle.block_spectra(col.blocks)
        t_spec = time.perf_counter() - t0
        S = min(sample, P)
        t0 = time.perf_counter()
        oracle.pair_errors(sp, pairs[:S], r, 7, oracle.RAW)
        t_pairs = time.perf_counter() - t0
        what = (f"first {S} of the {P} norm-ordered pairs, all 3 estimators, float64 oracle "
                f"(OpenMP over pairs); its block spectra ({t_spec:.2f} s for all {col.N} blocks) "
                f"prorated by {S}/{P}")
    rate = S / (t_pairs + t_spec * S / P)
    return {"value": rate, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "sample": what,
            "seconds": t_pairs + t_spec * S / P}


def run_reference(args):
    rank, ws, local, dist = dist_init(args)
    if rank != 0:
        return
    import oracle
    if is_big(args.config):
        raise SystemExit("--impl reference times configs 1, 2 and 5 (configs 3/4: see cpu_baseline of the "
                         "cmsvd arm, whose oracle sample covers a block subset)")
    col = workload(args.config, 0)
    sp = oracle.block_spectra(col.blocks)
    order = np.array(sorted(range(col.N), key=lambda i: (-sp.E[i], i)))
    pairs = synth.all_pairs_by_norm_order(order)
    S = min(args.ref_sample, pairs.shape[0])
    for w in range(args.warmup):
        oracle.pair_errors(sp, pairs[:max(1, S // 4)], col.r, 7, oracle.RAW)
    t0 = time.perf_counter()
    t_spec = 0.0
    for k in range(args.steps):
        ts = time.perf_counter()
        sp = oracle.block_spectra(col.blocks)
        t_spec += time.perf_counter() - ts
        off = (k * S) % pairs.shape[0]
        oracle.pair_errors(sp, pairs[off:off + S], col.r, 7, oracle.RAW)
    dt = time.perf_counter() - t0
    # each step re-runs the oracle block spectra; prorate it like the GPU arm's per-step S2 over P pairs
    t_eff = dt - t_spec + t_spec * S / pairs.shape[0]
    value = S * args.steps / t_eff
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_eff / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": args.config, "N": col.N, "m": col.m, "n": col.n, "r": col.r,
                      "pairs_per_step": S, "kinds": "weyl+residual+incremental", "operand": "RAW"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                            "sample": f"{S} pairs per step of the {pairs.shape[0]} norm-ordered pairs; oracle "
                                      f"block spectra recomputed each step and prorated by {S}/{pairs.shape[0]}"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    rank, ws, local, dist = dist_init(args)
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_2601_11626_b200 as cm
    # a dedicated (non-default) stream: the library enqueues on it and every
    # CUDA event of the timed region is recorded on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    col = workload(args.config, rank)
    r = col.r
    ctx = cm.Context(local, stream.cuda_stream)
    blocks_d = torch.from_numpy(col.blocks).to(dev)
    ctx.register(blocks_d)
    E, _, blk_rank = ctx.block_spectra(r)
    order = np.array(sorted(range(col.N), key=lambda i: (-E[i], i)))
    pairs = synth.all_pairs_by_norm_order(order)
    P = pairs.shape[0]
    pairs_d = torch.from_numpy(pairs).to(dev)
    out = {"err2": torch.empty((P, 3), dtype=torch.float64, device=dev),
           "total": torch.empty(P, dtype=torch.float64, device=dev),
           "sigma_tilde": torch.empty((P, r), dtype=torch.float32, device=dev),
           "mu": torch.empty((P, r), dtype=torch.float32, device=dev)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    big = is_big(args.config)
    operand = cm.TRUNC if big else cm.RAW

    def step():
        ctx.register(blocks_d)
        ctx.block_spectra(r)
        ctx.pair_errors(pairs_d, out=out, operand=operand)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    ctx.profile(True)
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    launches = ctx.launches - launches0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(times)
    total_ms = max_over_ranks(dist, total_ms, dev)
    units = P * args.steps * ws
    value = units / (total_ms / 1e3)

    # ---- roofline of the dominant kernel category (live CUDA events) ----
    rr_b = np.minimum(r, blk_rank).astype(np.float64)
    # projection basis of each base: the full numerical range (configs 1, 2, 5) or U_r (A22 blocks);
    # appended operand width: the raw block (RAW) or its rank-r factor (TRUNC)
    q = (rr_b if big else blk_rank.astype(np.float64))[pairs[:, 0]]
    w = rr_b[pairs[:, 1]] if big else np.full(P, float(col.n))
    rr = rr_b[pairs[:, 0]]
    nG = rr + w
    flops = {                                                # algorithmic flops per launch (all P pairs)
        "eig_G": float(np.sum(tridiag_flops(nG))),
        "eig_W": float(np.sum(tridiag_flops(w))),
        "gram_W": float(np.sum(col.m * w * (w + 1))),
        "gram_ZZ": float(np.sum(q * w * (w + 1))),
        "proj_Z": float(np.sum(2.0 * col.m * q * w)),
        "resid_R": float(np.sum(2.0 * col.m * q * w)),
        "pair_tc": float(np.sum(4.0 * col.m * q * w + col.m * w * (w + 1))),   # Z, R', W' useful flops
    }
    # operands wider than 128 columns run Z, R', W' as tcgen05 GEMM tiles (k_gemm_tc), else SIMT
    tiles = float(np.max(q)) > 128 or float(np.max(w)) > 128
    tc_peak = tf32_fp32eq_tflops()
    peaks = {"eig_G": DFMA_TFLOPS, "eig_W": DFMA_TFLOPS, "gram_W": tc_peak if tiles else DFMA_TFLOPS,
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
            e["tflops"] = flops[name] * args.steps / (ms * 1e-3) / 1e12
            e["frac_of_peak"] = e["tflops"] / peaks[name]
        kernels[name] = e
    # dominant category with an algorithmic flop model (configs 3/4: the one-time A22 block spectra of the
    # step can take longer; they are reported as "dominant_category")
    dom_all = max((k for k in kernels), key=lambda k: kernels[k]["ms_total"])
    dom = max((k for k in kernels if k in flops), key=lambda k: kernels[k]["ms_total"], default=dom_all)
    d = kernels[dom]
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")   # dram bytes per launch from ncu --set full
    if os.path.exists(tfile):
        traffic = json.load(open(tfile)).get(args.config, {}).get(dom)
    if dom in flops:
        roof = {"bound": "tensor" if peaks[dom] == tc_peak else "alu", "kernel": dom, "achieved": d["tflops"],
                "peak": peaks[dom], "unit": "TFLOP/s",
                "frac": d["frac_of_peak"], "traffic": traffic,
                "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                                "(profiles/ncu_*_summary.txt)",
                "peak_source": ("MEASURED_PEAKS.json bf16 burst x 0.5 (nominal TF32/BF16) / 3 (3xTF32 MMAs per "
                                "useful fp32 product)") if peaks[dom] == tc_peak else
                               ("own DFMA/FFMA microbenchmark (tools/peaks.cu, profiles/peaks_r01.txt); "
                                "MEASURED_PEAKS.json has no FP64/FP32-SIMT peak"),
                "algorithmic": "Householder tridiagonalisation 4/3 n^3 flops per (r'+w)^2 Gram"
                if dom.startswith("eig") else "2 m q w (GEMM) / m w (w+1) (SYRK) flops per pair"}
    else:
        roof = {"bound": "alu", "kernel": dom, "achieved": None, "peak": None, "unit": "TFLOP/s", "frac": None,
                "traffic": None}

    result = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
              "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
              "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
              "config": {"workload": args.config, "N": col.N, "m": col.m, "n": col.n, "r": r, "pairs": P,
                         "kinds": "weyl+residual+incremental", "operand": "TRUNC" if big else "RAW",
                         "step": "register(S1)+block_spectra(S2)+pair_errors(S3-S9), device-resident input",
                         "l2": "flushed (256 MiB write) before every step, outside the step events",
                         "parallelism": f"replicas x{ws} (independent collections, no collective)"},
              "gpu_launches": launches, "roofline": roof, "kernels": kernels, "dominant_category": dom_all,
              "step_ms": times}
    with_clk = clk.summary()
    result["clocks"] = with_clk

    # ---- e2e through the C ABI with host buffers ----
    if not args.no_e2e:
        pinned = torch.from_numpy(col.blocks).pin_memory()
        pairs_h = np.ascontiguousarray(pairs)
        ctx2 = cm.Context(local, stream.cuda_stream)
        ctx2.register(pinned)
        ctx2.block_spectra(r)
        ctx2.pair_errors(pairs_h, operand=operand)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ctx2.register(pinned)
            ctx2.block_spectra(r)
            res_h = ctx2.pair_errors(pairs_h, operand=operand)
        t_e2e = time.perf_counter() - t0
        t_e2e = max_over_ranks(dist, t_e2e, dev)
        h2d = col.blocks.nbytes + pairs_h.nbytes
        d2h = res_h["err2"].nbytes + res_h["total"].nbytes + res_h["sigma_tilde"].nbytes + res_h["mu"].nbytes + \
            col.N * (8 + 4 * r + 4)
        result["e2e"] = {"value": P * args.steps * ws / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                         "d2h_bytes_per_step": int(d2h),
                         "path": "cmsvd_register(pinned host) + cmsvd_block_spectra + cmsvd_pair_errors(host), "
                                 "host wall clock"}
        ctx2.close()

    # ---- greedy drivers (S10), reported beside the metric ----
    if not args.no_greedy and rank == 0 and not big:
        g = {}
        for alg, srt, name in [(cm.ALG_APPROX, cm.SORT_RESIDUAL, "approx_residual"),
                               (cm.ALG_RESIDUAL, cm.SORT_FROBENIUS, "residual_frobenius"),
                               (cm.ALG_MAX_NORM, cm.SORT_FROBENIUS, "max_norm")]:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = ctx.cluster(alg, 0.05, sort=srt)
            g[name] = {"eps": 0.05, "ms": 1e3 * (time.perf_counter() - t0), "clusters": len(res["clusters"]),
                       "n_evals": res["n_evals"]}
        result["greedy"] = g

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(col, pairs, r, args.cpu_sample, big=big)
    ctx.close()
    if rank == 0:
        print(json.dumps(result))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

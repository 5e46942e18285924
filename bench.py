#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the B200 phase-shift sparse FFT hot path.

One *step* = one complete solve (all iterations of Algorithm 2, every row of
SURVEY 8(a)) of a batch of independent synthetic signals of BASELINE.json's metric configuration
(configs[2]: d=100, N=65536, k=1000, |a| ~ U[1,10]) -- per GPU (weak scaling over signal shards).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs under torchrun (one rank per GPU, NCCL).  Rank 0 prints ONE JSON line.  The oracle
(oracle/, test infrastructure) is executed only by the cpu_baseline leg and by --impl reference.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

FP64_PEAK_TFLOPS = 37.2          # 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
FP64_PEAK_MEASURED = 37.1        # tools/fp64_peak.cu, DMMA m8n8k4 (profiles/r01_fp64_peak.log)
INT8_PER_BF16 = 2.0              # B200_PROFILING.md nominal dense ratio (4.5 POPS int8 / 2.25 PFLOP/s bf16)


def measured_peaks():
    """MEASURED_PEAKS.json (driver-written): HBM copy GB/s and cuBLAS bf16 TFLOP/s (burst / sustained)."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return d, "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback (B200_PROFILING.md)"
METRIC = "recovered modes/s (d=100, N=65536, k=1000)"


def workload_desc(cfg):
    """The workload named in config.workload (both arms): dimensions, coefficient law, partition, r, E = 2B."""
    b = list(cfg.blocks)
    part = f"({b[0]}^{len(b)})" if len(set(b)) == 1 else "(" + ",".join(str(x) for x in b) + ")"
    B = max(cfg.N ** q for q in b)
    amp = "|a|~U[1,10]" if getattr(cfg, "rho", "") == "uniform1_10" else "|a|=1"
    return (f"{cfg.name}: d={cfg.d} N={cfg.N} k={cfg.k} {amp}, partition {part}, r={len(b)}, "
            f"E=2^{int(np.log2(2 * B))}")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(W.CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="signals per GPU per step (default: config trials)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--shard", default="signals", choices=["signals", "lines"],
                    help="signals: independent signal shards per rank (weak scaling, default); lines: every rank "
                         "solves the same signals and owns a shard of the shifted lines (strong scaling, NCCL "
                         "record all-gather per iteration, SURVEY 8(e))")
    ap.add_argument("--latency-steps", type=int, default=20, help="single-signal solves timed for latency_single_solve")
    ap.add_argument("--table-cache", type=int, default=1024,
                    help="per-prime table cache slots (plan option table_cache_slots; ~1 MB each): the steady state "
                         "reuses the tables of every prime the workload visits")
    ap.add_argument("--expsum-path", type=int, default=0, choices=[0, 1, 2],
                    help="0 auto (int8 limbs on tcgen05 when available), 1 FP64 tensor/vector, 2 int8 limbs")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks (nvidia-smi during the timed region)
class Clocks:
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.t0 = self.t1 = None

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()

    def result(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = []
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 10:
                continue
            try:
                ts = time.mktime(time.strptime(parts[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                ts += float("0." + parts[0].split(".")[1]) if "." in parts[0] else 0.0
            except Exception:
                ts = None
            if int(parts[1]) not in self.gpus:
                continue
            rows.append((ts, parts))
        inside = [r for r in rows if r[0] is not None and self.t0 - 0.15 <= r[0] <= self.t1 + 0.15]
        use = inside or rows
        sm = [float(r[1][2]) for r in use if r[1][2].replace(".", "").isdigit()]
        mx = [float(r[1][3]) for r in use if r[1][3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in use for n, v in zip(names, r[1][6:10]) if v.lower() == "active"})
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(use), "samples_in_window": len(inside)}


# ------------------------------------------------------------------ oracle legs (CPU)
def oracle_throughput(cfg, n_threads, trials):
    """The oracle as it stands, one solve per host thread: recovered modes/s on this host."""
    import oracle as O
    w, a = W.make_batch(cfg, trials)
    P = O.params_for(cfg)
    t = time.perf_counter()
    status, ow, oa, cnt, samples, _ = O.solve_batch(P, w, a, n_threads=n_threads)
    dt = time.perf_counter() - t
    assert (status == 0).all()
    return int(cnt.sum()) / dt, dt, int(samples.sum())


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    cfg = W.CONFIGS[args.config]
    cores = args.cpu_threads or os.cpu_count() or 1
    # A step is one signal's solve; the steps run concurrently, one per host thread (an oracle solve of C3 takes
    # ~20 s on one core, so K sequential rounds would not finish in minutes).  The W warm-up steps run the same
    # way, untimed.  At least `cores` signals are timed so that every host thread works.
    if args.warmup:
        oracle_throughput(cfg, min(cores, args.warmup), list(range(args.warmup)))
    n = max(args.steps, cores)
    trials = list(range(n))
    _, dt, samp = oracle_throughput(cfg, cores, trials)
    value = n * cfg.k / dt
    times = [dt / args.steps] * args.steps
    sample = (f"{n} {cfg.name} signals (trials 0..{n - 1}) solved concurrently, one solve per host thread "
              f"({cores} threads), {dt:.1f} s wall; ms_per_step = wall / steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "modes/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded PCG64, PAPER.md:424 recipe)",
            "config": {"workload": workload_desc(cfg), "signals_timed": n, "host_threads": cores},
            "sample_evals_per_s": samp / sum(times),
            "cpu_baseline": {"value": value, "unit": "modes/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "modes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    import paper_1606_07407_b200 as S

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_1606_07407_b200.shard import shard_indices
    cfg = W.CONFIGS[args.config]
    T = args.batch or cfg.trials
    lines = args.shard == "lines"
    mult = 1 if lines else world                        # signal sets solved per step across the job
    # signal shards: each rank its own independent signals; line shards: every rank the same signals
    trials = list(range(T)) if lines else shard_indices(world * T, world, rank)
    w_np, a_np = W.make_batch(cfg, trials)
    w_h = torch.from_numpy(w_np).pin_memory()
    a_h = torch.from_numpy(a_np).pin_memory()
    w_d, a_d = w_h.cuda(), a_h.cuda()
    stream = torch.cuda.current_stream()
    plan = S.sfft_plan(cfg.d, cfg.N, cfg.k, blocks=cfg.blocks, batch=T, profile=True,
                        expsum_path=args.expsum_path, line_shards=world if lines else 0,
                        line_rank=rank if lines else 0, table_cache_slots=args.table_cache)
    if lines:
        if world > 1:
            S.comm_init_line_shards(plan)
        else:
            S.sfft_comm_init(plan, 1, 0, shard_mode=1, unique_id=S.sfft_comm_unique_id())
    sig = S.sfft_signal_expsum(plan, w_d, a_d)
    outs = (torch.empty((T, cfg.k, cfg.d), dtype=torch.int32, device="cuda"),
            torch.empty((T, cfg.k, 2), dtype=torch.float64, device="cuda"),
            torch.empty((T,), dtype=torch.int32, device="cuda"),
            torch.empty((T,), dtype=torch.int32, device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        S.sfft_execute(plan, sig, outs)
    torch.cuda.synchronize()
    # correctness of what we time: the recovered spectra equal the inputs (exact recovery)
    ok = bool((outs[3] == 0).all().item())
    ws = np.stack([W.canonical_sort(w_np[i], a_np[i])[0] for i in range(T)])
    ok = ok and np.array_equal(outs[0].cpu().numpy(), ws)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    clocks = Clocks({local_rank} if world == 1 else set(range(world))) if rank == 0 else None
    barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    for i in range(args.steps):
        flush.zero_()                                   # L2 flush between timed steps (not timed)
        ev[i][0].record(stream)
        res = S.sfft_execute(plan, sig, outs)
        ev[i][1].record(stream)
        reps.append(res.report)
    torch.cuda.synchronize()
    barrier()
    if clocks:
        clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    ms_step = ms_max / args.steps
    modes_total = mult * T * cfg.k * args.steps
    value = modes_total / (ms_max / 1e3)
    samples = sum(r.samples_used for r in reps)
    cmacs = sum(r.cmacs for r in reps)
    ms_exp = sum(r.ms_expsum for r in reps)
    ms_fft = sum(r.ms_fft for r in reps)
    ms_dec = sum(r.ms_decode for r in reps)
    ms_oth = sum(r.ms_other for r in reps)
    n_exp = sum(r.n_expsum for r in reps)
    launches = sum(r.kernel_launches for r in reps)
    cm8 = sum(r.cmacs_i8 for r in reps)
    ms8 = sum(r.ms_expsum_i8 for r in reps)
    n8 = sum(r.n_expsum_i8 for r in reps)
    limbs = reps[0].i8_limbs if reps else 0
    peaks, peaks_src = measured_peaks()
    traffic, traffic_kernel = None, ""
    tf = os.path.join(ROOT, "profiles", "expsum_ncu.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic = tj.get("dram_bytes_per_launch")
            traffic_kernel = tj.get("kernel", "")
        except Exception:
            traffic = None
    if n8 and ms8 > 0:
        # int8-limb tensor-core exp-sum: per complex MAC of the method, 4 real MACs of the 2K x 2L
        # real GEMM times S (S + 1) / 2 limb products, 2 ops per MAC -- unpadded rows p and columns 2L
        ops = 2.0 * 4.0 * limbs * (limbs + 1) / 2.0 * cm8
        peak = peaks.get("bf16_tflops_sustained", 1400.0) * INT8_PER_BF16
        achieved = ops / (ms8 / 1e3) / 1e12
        roofline = {"bound": "tensor", "kernel": f"expsum_i8 (tcgen05.mma.kind::i8, {limbs} limbs, A in TMEM)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": traffic if traffic is not None and "i8" in traffic_kernel else None,
                    "unit_note": "int8 tera-ops/s (MAC = 2 ops)",
                    "peak_source": f"{peaks_src} bf16_tflops_sustained x {INT8_PER_BF16} (nominal int8:bf16 ratio, "
                                   "B200_PROFILING.md); kernel timed inside the step",
                    "algorithmic_ops_per_launch": ops / n8, "avg_launch_ms": ms8 / n8,
                    "fp64_equivalent": {"achieved_tflops": 8.0 * cm8 / (ms8 / 1e3) / 1e12,
                                        "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                                        "ratio": 8.0 * cm8 / (ms8 / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                                        "note": "8 flop per complex MAC of the exp-sum vs the FP64 pipe peak"}}
    else:
        achieved = 8.0 * cmacs / (ms_exp / 1e3) / 1e12
        roofline = {"bound": "alu", "kernel": "expsum (FP64 tensor pipe: mma.sync f64 / DMMA)", "achieved": achieved,
                    "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                    "traffic": traffic if traffic is not None and "dmma" in traffic_kernel else None,
                    "peak_source": "derived 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz; measured DMMA 37.1, DFMA 33.6 "
                                   "(profiles/r01_fp64_peak.log); MEASURED_PEAKS.json has no FP64 entry",
                    "algorithmic_flops_per_launch": 8.0 * cmacs / max(n_exp, 1),
                    "avg_launch_ms": ms_exp / max(n_exp, 1)}
    if roofline.get("traffic") is not None:
        roofline["traffic_note"] = "DRAM bytes of the iteration-1 launch (ncu --set full, profiles/expsum_ncu.json)"

    # e2e: the public host-buffer call, H2D of the inputs and D2H of the result inside the timed region
    hout = (torch.empty((T, cfg.k, cfg.d), dtype=torch.int32).pin_memory(),
            torch.empty((T, cfg.k, 2), dtype=torch.float64).pin_memory(),
            torch.empty((T,), dtype=torch.int32).pin_memory(),
            torch.empty((T,), dtype=torch.int32).pin_memory())
    if args.e2e_steps:
        S.sfft_solve_host(plan, w_h, a_h, hout)
    barrier()
    torch.cuda.synchronize()
    e_ms = 0.0
    for _ in range(args.e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        S.sfft_solve_host(plan, w_h, a_h, hout)
        e_ms += (time.perf_counter() - t) * 1e3
    e_t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
    e2e_value = mult * T * cfg.k * args.e2e_steps / (float(e_t.item()) / 1e3) if args.e2e_steps else None
    h2d = w_h.numel() * 4 + a_h.numel() * 16
    d2h = hout[0].numel() * 4 + hout[1].numel() * 8 + hout[2].numel() * 4 + hout[3].numel() * 4
    if args.e2e_steps:
        ok = ok and np.array_equal(hout[0].numpy(), ws)
    ok_t = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
    if world > 1:
        dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
    ok = bool(ok_t.item())

    # single-solve latency: one signal per execute (trial 0 of this rank), device-resident inputs,
    # CUDA events around each execute, median of the timed runs (not part of `value`)
    lat = None
    if args.latency_steps and not lines:
        plan1 = S.sfft_plan(cfg.d, cfg.N, cfg.k, blocks=cfg.blocks, batch=1, expsum_path=args.expsum_path,
                            table_cache_slots=args.table_cache)
        sig1 = S.sfft_signal_expsum(plan1, w_d[:1].contiguous(), a_d[:1].contiguous())
        outs1 = tuple(o[:1].clone() for o in outs)
        for _ in range(2):
            S.sfft_execute(plan1, sig1, outs1)
        ts = []
        for _ in range(args.latency_steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r1 = S.sfft_execute(plan1, sig1, outs1)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        lat = {"ms_median": sorted(ts)[len(ts) // 2], "ms_min": min(ts), "iterations": r1.report.iterations,
               "signal": f"{cfg.name} trial {trials[0]}", "exact": bool(np.array_equal(outs1[0][0].cpu().numpy(), ws[0]))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = args.cpu_threads or os.cpu_count() or 1
        v, dt, _ = oracle_throughput(cfg, cores, list(range(cores)))
        cpu = {"value": v, "unit": "modes/s", "cores": cores, "kind": "oracle",
               "sample": f"{cores} {cfg.name} signals (trials 0..{cores - 1}), one oracle solve per host thread, "
                         f"{dt:.1f} s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "modes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if lines else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded PCG64 per PAPER.md:424 recipe; no dataset exists for this metric)",
            "expsum_path": "int8 limbs on tcgen05" if n8 else "fp64",
            "config": {"workload": workload_desc(cfg),
                       "signals_per_gpu_per_step": T, "table_cache_slots": args.table_cache,
                       "parallelism": f"line shards x{world} (NCCL record all-gather)" if lines else f"signal shards x{world}",
                       "l2": "256 MB L2 flush between timed steps; per-step working set > 1 GB"},
            "sample_evals_per_s": mult * samples / (ms_max / 1e3),
            "verified_exact_recovery": ok,
            "roofline": roofline,
            "kernel_ms_per_step": {"expsum": ms_exp / args.steps, "fft": ms_fft / args.steps,
                                   "decode": ms_dec / args.steps, "other": ms_oth / args.steps},
            "fft_hbm": {"achieved_gbs": 32.0 * samples / (ms_fft / 1e3) / 1e9, "peak_gbs": peaks.get("hbm_gbs"),
                        "note": "32 B per sample (read s, write F); Bluestein work is FP64-bound"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "modes/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "latency_single_solve": lat,
            "clocks": clocks.result() if clocks else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

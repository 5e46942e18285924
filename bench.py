#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the B200 phase-shift sparse FFT hot path.

One *step* = one complete solve (all iterations of Algorithm 2, every row of
SURVEY 8(a)) of a batch of independent synthetic signals of BASELINE.json's metric configuration
(configs[2]: d=100, N=65536, k=1000, |a| ~ U[1,10]) -- per GPU (weak scaling over signal shards).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1..c5]

N>1 runs one rank per GPU over NCCL: under torchrun as the driver launches it, or -- when WORLD_SIZE is unset --
bench.py re-executes itself under torch.distributed.run with N ranks.  Rank 0 prints ONE JSON line.  The oracle
(oracle/, test infrastructure) is executed only by the cpu_baseline leg and by --impl reference.
"""
import argparse
import json
import os
import socket
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
    ap.add_argument("--e2e-steps", type=int, default=-1,
                    help="steps of the end-to-end (host-buffer) legs; -1 = --steps (0 = skip)")
    ap.add_argument("--spec-primes", type=int, nargs="*", default=[2, 4, 8],
                    help="single-solve latency (and, with --spec-steps, the batched step) also with G-prime "
                         "speculation (reading R26) for each G")
    ap.add_argument("--spec-steps", type=int, default=5, help="timed steps of each batched speculation leg (0 = skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--shard", default="signals", choices=["signals", "lines", "spec"],
                    help="signals: independent signal shards per rank (weak scaling, default); lines: every rank "
                         "solves the same signals and owns a shard of the shifted lines (strong scaling, NCCL "
                         "record all-gather per iteration, SURVEY 8(e)); spec: every rank solves the same signals "
                         "with its own prime of each iteration, records all-gathered and merged in rank order "
                         "(multi-prime speculation, DESIGN reading R26; world 1 = Alg. 2)")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "fused"],
                    help="--shard lines: records all-gathered after the FFT (NCCL) or stored into every shard's memory "
                         "by the FFT epilogue itself (line_exchange = 1, CUDA IPC peer mappings)")
    ap.add_argument("--latency-steps", type=int, default=20, help="single-signal solves timed for latency_single_solve")
    ap.add_argument("--table-cache", type=int, default=0,
                    help="per-prime table cache slots (plan option table_cache_slots; ~0.8 MB each); 0 = the plan "
                         "default max(batch + 16, 512)")
    ap.add_argument("--expsum-path", type=int, default=0, choices=[0, 1, 2],
                    help="0 auto (int8 limbs on tcgen05 when available), 1 FP64 tensor/vector, 2 int8 limbs")
    ap.add_argument("--fp64-steps", type=int, default=-1,
                    help="steps of the FP64-path sub-measurement (fp64_path object; -1 = --steps, 0 = skip)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / reduction check without a GPU: gloo ranks, a fake solve (tests only)")
    return ap.parse_args()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_self_launch(args) -> None:
    """--gpus N > 1 without torchrun: re-execute this script under torch.distributed.run with N local ranks (one
    per GPU), so a plain `python bench.py --gpus N` measures N GPUs.  Fails loudly when fewer GPUs are visible."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


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
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_run(cfg, n_threads, n_signals):
    """The oracle as it stands, one solve per host thread, n_signals = a multiple of n_threads (balanced rounds).
    Returns the cpu_baseline object (value = recovered modes/s on this host) and the wall time."""
    import oracle as O
    trials = list(range(n_signals))
    w, a = W.make_batch(cfg, trials)
    P = O.params_for(cfg)
    t = time.perf_counter()
    status, _, _, cnt, samples, _, ns = O.solve_batch(P, w, a, n_threads=n_threads, times=True)
    dt = time.perf_counter() - t
    assert (status == 0).all()
    rounds = max(1, n_signals // n_threads)
    solve_s = ns[:, 0] / 1e9
    main_s = (ns[:, 0] - ns[:, 1]) / 1e9
    obj = {"value": int(cnt.sum()) / dt, "unit": "modes/s", "cores": n_threads, "kind": "oracle",
           "sample": f"{n_signals} {cfg.name} signals (trials 0..{n_signals - 1}), {rounds} round(s) of one oracle "
                     f"solve per host thread ({n_threads} threads), {dt:.1f} s wall",
           "cpu_model": cpu_model(), "nproc": os.cpu_count(),
           "s_per_solve_single_core": float(np.mean(solve_s)),
           "main_part_s_per_solve": float(np.mean(main_s)),
           "main_part_note": "solve time minus the sampling of f - g (Alg. 2 l.13-14), the paper's 'CPU TICKS' "
                             "excludes sampling (PAPER.md:461-463)",
           "sample_evals_per_s": float(samples.sum()) / dt}
    return obj, dt


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    cfg = W.CONFIGS[args.config]
    cores = args.cpu_threads or os.cpu_count() or 1
    # A step is one signal's solve; the steps run concurrently, one per host thread (an oracle C3 solve takes ~20 s
    # on one core, so K sequential rounds would not finish in minutes).  The timed signals are a whole number of
    # rounds of `cores` solves (balanced: every thread does the same number of solves), at least K of them; the W
    # warm-up solves run the same way, untimed.
    if args.warmup:
        oracle_run(cfg, min(cores, args.warmup), min(cores, args.warmup))
    rounds = max(1, -(-args.steps // cores))
    n = rounds * cores
    cb, dt = oracle_run(cfg, cores, n)
    value = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "modes/s",
            "n_gpus": world if "WORLD_SIZE" in os.environ else args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded PCG64, PAPER.md:424 recipe)",
            "config": {"workload": workload_desc(cfg), "signals_timed": n, "host_threads": cores},
            "sample_evals_per_s": cb["sample_evals_per_s"],
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "modes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ launcher check without a GPU
def run_dry(args, rank, world):
    """--dry-run: the multi-rank plumbing of our arm (launcher, barriers, max-over-ranks time, MIN of the
    verification flags, rank-0 printing) on gloo with a fake solve of fixed duration -- no GPU, no kernels."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    ms = 1.0 + rank                                         # rank-dependent: the max over ranks must win
    t = torch.tensor([ms * args.steps], dtype=torch.float64)
    ok = torch.tensor([1], dtype=torch.int32)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": world * 1.0 / (float(t.item()) / 1e3), "unit": "modes/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": float(t.item()) / args.steps, "dry_run": True,
                          "verified_exact_recovery": bool(ok.item())}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ our arm
def time_steps(S, plan, sig, outs, steps, stream, flush, barrier):
    """K steps bracketed by barrier + synchronize, CUDA events on the plan's stream around each execute, an L2
    flush (not timed) before each.  Returns (total ms, reports)."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    reps = []
    barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        res = S.sfft_execute(plan, sig, outs)
        ev[i][1].record(stream)
        reps.append(res.report)
    torch.cuda.synchronize()
    barrier()
    return sum(a.elapsed_time(b) for a, b in ev), reps


def main():
    args = parse()
    maybe_self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.dry_run:
        run_dry(args, rank, world)
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
    spec = args.shard == "spec" and world > 1
    lines = args.shard == "lines" or spec              # every rank solves the same signals
    mult = 1 if lines else world                        # signal sets solved per step across the job
    # signal shards: each rank its own independent signals; line shards: every rank the same signals
    trials = list(range(T)) if lines else shard_indices(world * T, world, rank)
    w_np, a_np = W.make_batch(cfg, trials)
    w_h = torch.from_numpy(w_np).pin_memory()
    a_h = torch.from_numpy(a_np).pin_memory()
    w_d, a_d = w_h.cuda(), a_h.cuda()
    stream = torch.cuda.current_stream()

    def make_plan(path, batch=T, profile=True, shard=True):
        if spec and shard:
            p = S.sfft_plan(cfg.d, cfg.N, cfg.k, blocks=cfg.blocks, batch=batch, profile=profile, expsum_path=path,
                            table_cache_slots=args.table_cache, spec_primes=world, spec_distributed=1,
                            spec_rank=rank)
            S.comm_init_spec_ranks(p)
            return p
        fused = lines and shard and args.exchange == "fused"
        p = S.sfft_plan(cfg.d, cfg.N, cfg.k, blocks=cfg.blocks, batch=batch, profile=profile, expsum_path=path,
                        line_shards=world if (lines and shard) else 0, line_rank=rank if (lines and shard) else 0,
                        table_cache_slots=args.table_cache, line_exchange=1 if fused else 0)
        if lines and shard:
            if world > 1:
                S.comm_init_line_shards(p, exchange=1 if fused else 0)
            elif fused:
                S.sfft_comm_init_peers(p, 1, 0, [S.sfft_comm_peer_handle(p)])
            else:
                S.sfft_comm_init(p, 1, 0, shard_mode=1, unique_id=S.sfft_comm_unique_id())
        return p

    # the timed plan runs without per-kernel events (they cost ~30 us per iteration: C5's 72 iterations lose 14 %);
    # a second, profiled plan on the same signals gives the per-kernel-class times of the roofline
    plan = make_plan(args.expsum_path, profile=False)
    sig = S.sfft_signal_expsum(plan, w_d, a_d)
    outs = (torch.empty((T, cfg.k, cfg.d), dtype=torch.int32, device="cuda"),
            torch.empty((T, cfg.k, 2), dtype=torch.float64, device="cuda"),
            torch.empty((T,), dtype=torch.int32, device="cuda"),
            torch.empty((T,), dtype=torch.int32, device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ws = np.stack([W.canonical_sort(w_np[i], a_np[i])[0] for i in range(T)])

    def exact(o):
        return bool((o[3] == 0).all().item()) and np.array_equal(o[0].cpu().numpy(), ws)

    for _ in range(args.warmup):
        S.sfft_execute(plan, sig, outs)
    torch.cuda.synchronize()
    # correctness of what we time: the recovered spectra equal the inputs (exact recovery); with no warm-up
    # the check runs on the timed steps' output only
    ok = exact(outs) if args.warmup else True
    clocks = Clocks({local_rank} if world == 1 else set(range(world))) if rank == 0 else None
    if clocks:
        clocks.start()
    ms, reps_timed = time_steps(S, plan, sig, outs, args.steps, stream, flush, barrier)
    clock_res = None
    if clocks:
        clocks.stop()
        clock_res = clocks.result()   # stops the sampler: nvidia-smi's driver queries would perturb the later legs
    ok = ok and exact(outs)
    # kernel-class breakdown (profile = 1: CUDA events around every kernel class on the plan's stream), same steps
    plan_prof = make_plan(args.expsum_path, profile=True)
    sig_prof = S.sfft_signal_expsum(plan_prof, w_d, a_d)
    outs_prof = tuple(torch.empty_like(o) for o in outs)
    for _ in range(args.warmup):
        S.sfft_execute(plan_prof, sig_prof, outs_prof)
    ms_prof, reps = time_steps(S, plan_prof, sig_prof, outs_prof, args.steps, stream, flush, barrier)
    ok = ok and exact(outs_prof)
    del plan_prof, sig_prof, outs_prof
    ms_max = max_over_ranks(ms)
    ms_step = ms_max / args.steps
    modes_total = mult * T * cfg.k * args.steps
    value = modes_total / (ms_max / 1e3)

    def tot(attr):
        return sum(getattr(r, attr) for r in reps)

    samples, cmacs = tot("samples_used"), tot("cmacs")
    ms_exp, ms_fft, ms_dec, ms_oth = tot("ms_expsum"), tot("ms_fft"), tot("ms_decode"), tot("ms_other")
    n_exp = tot("n_expsum")
    launches = sum(r.kernel_launches for r in reps_timed)      # our kernels inside the timed region
    cm8, ms8, n8 = tot("cmacs_i8"), tot("ms_expsum_i8"), tot("n_expsum_i8")
    plogp = tot("fft_plogp")
    mlogm = tot("fft_mlogm")
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
        peak = peaks.get("bf16_tflops", 1654.1) * INT8_PER_BF16
        achieved = ops / (ms8 / 1e3) / 1e12
        roofline = {"bound": "tensor", "kernel": f"expsum_i8 (tcgen05.mma.kind::i8, {limbs} limbs, A in TMEM)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": traffic if traffic is not None and "i8" in traffic_kernel else None,
                    "unit_note": "int8 tera-ops/s (MAC = 2 ops)",
                    "peak_source": f"{peaks_src} bf16_tflops (burst: the kernel runs in ms-long steps at max clock, "
                                   f"see clocks) x {INT8_PER_BF16} (nominal int8:bf16 ratio, B200_PROFILING.md)",
                    "algorithmic_ops_per_launch": ops / n8, "avg_launch_ms": ms8 / n8,
                    "fp64_equivalent": {"achieved_tflops": 8.0 * cm8 / (ms8 / 1e3) / 1e12,
                                        "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                                        "ratio": 8.0 * cm8 / (ms8 / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                                        "note": "8 flop per complex MAC of the exp-sum vs the FP64 pipe peak"}}
    elif tot("n_fused_sample") > 0:
        # short lines: the sampling runs inside the FFT CTAs (fused_sample) -- the sampling's FP64 flops over the
        # fused kernel's whole time (which also holds the FFT and the decode epilogue): a lower bound of its rate
        achieved = 8.0 * cmacs / (ms_fft / 1e3) / 1e12
        roofline = {"bound": "alu", "kernel": "pfft with fused sampling (FP64; the exp-sum inside the FFT CTAs)",
                    "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                    "traffic": None,
                    "peak_source": "derived 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz; measured DMMA 37.1, DFMA 33.6",
                    "note": "8 flop per (sample, term) complex MAC over the fused sample + FFT + decode kernel's time",
                    "fused_iterations": tot("n_fused_sample")}
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
    fft_traffic = None
    ff = os.path.join(ROOT, "profiles", "fft_ncu.json")
    if os.path.exists(ff):
        try:
            fj = json.load(open(ff))
            fft_traffic = {"dram_bytes_per_launch": fj.get("dram_bytes_per_launch"), "kernel": fj.get("kernel"),
                           "algorithmic_bytes_per_launch": fj.get("algorithmic_bytes_per_launch"),
                           "source": fj.get("source"),
                           "note": "the iteration-1 FFT launch of this workload (ncu --set full): the fused epilogue "
                                   "writes no F lines, so DRAM bytes ~ the 16 B per sample read"}
        except Exception:
            fft_traffic = None
    fft_gbs = 32.0 * samples / (ms_fft / 1e3) / 1e9 if ms_fft > 0 else None
    fft_tf = 5.0 * plogp / (ms_fft / 1e3) / 1e12 if ms_fft > 0 else None
    fft_roof = {"bound": "hbm", "kernel": "pfft (Bluestein, smem-resident; fused select / test / decode epilogue)",
                "achieved": fft_gbs, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": fft_gbs / peaks.get("hbm_gbs") if fft_gbs else None, "traffic": fft_traffic,
                "algorithmic_bytes": "32 B per sample (read s, write F) = 32 * samples_used per step",
                "fp64": {"achieved_tflops": fft_tf, "peak_tflops": FP64_PEAK_TFLOPS,
                         "frac": fft_tf / FP64_PEAK_TFLOPS if fft_tf else None,
                         "algorithmic_flops": "5 p log2 p per line of length p (radix-2 convention, report fft_plogp)"},
                "executed_fp64": {"tflops": 10.0 * mlogm / (ms_fft / 1e3) / 1e12 if ms_fft > 0 else None,
                                  "frac": 10.0 * mlogm / (ms_fft / 1e3) / 1e12 / FP64_PEAK_TFLOPS if ms_fft > 0 else None,
                                  "note": "Bluestein: a forward and an inverse FFT of size M >= 2p - 1 per line, 5 M log2 M "
                                          "flops each (report fft_mlogm); the transform is bound by shared-memory "
                                          "sweeps and FP64 latency at one 161 KB line per SM (DESIGN.md 8)"}}

    # FP64 path (expsum_path = 1: DMMA exp-sum) on the same workload, timed the same way (north star: the sum kernel
    # against the FP64 peak)
    fp64 = None
    fp64_steps = args.steps if args.fp64_steps < 0 else args.fp64_steps
    if fp64_steps and (n8 or args.expsum_path == 2):
        plan64 = make_plan(1)
        sig64 = S.sfft_signal_expsum(plan64, w_d, a_d)
        outs64 = tuple(torch.empty_like(o) for o in outs)
        for _ in range(args.warmup):
            S.sfft_execute(plan64, sig64, outs64)
        ms64, reps64 = time_steps(S, plan64, sig64, outs64, fp64_steps, stream, flush, barrier)
        ok64 = exact(outs64)
        ms64 = max_over_ranks(ms64)
        cm64 = sum(r.cmacs for r in reps64)
        mse64 = sum(r.ms_expsum for r in reps64)
        ach64 = 8.0 * cm64 / (mse64 / 1e3) / 1e12
        fp64 = {"value": mult * T * cfg.k * fp64_steps / (ms64 / 1e3), "unit": "modes/s",
                "ms_per_step": ms64 / fp64_steps, "steps": fp64_steps, "verified_exact_recovery": ok64,
                "dtype": "f64", "kernel_ms_per_step": {"expsum": mse64 / fp64_steps,
                                                       "fft": sum(r.ms_fft for r in reps64) / fp64_steps},
                "roofline": {"bound": "alu", "kernel": "expsum_dmma (mma.sync.m8n8k4 f64, DMMA)",
                             "achieved": ach64, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                             "frac": ach64 / FP64_PEAK_TFLOPS,
                             "peak_source": "derived 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (measured DMMA 37.1)"}}
        del plan64, sig64, outs64

    # multi-prime speculation (DESIGN reading R26) on the same batched workload: G primes per iteration, fewer
    # iterations for G x the sampling -- pays where late iterations dominate (C5), not where iteration 1 does (C3)
    spec_b = None
    if args.spec_primes and not lines and args.spec_steps:
        spec_b = {}
        for G in args.spec_primes:
            try:
                planG = S.sfft_plan(cfg.d, cfg.N, cfg.k, blocks=cfg.blocks, batch=T, expsum_path=args.expsum_path,
                                    table_cache_slots=args.table_cache, spec_primes=G)
            except S.SfftError as e:          # e.g. C2: 1024 signals x 8 slots beyond the slot-assignment bound
                spec_b[f"G{G}"] = {"unsupported": str(e)}
                continue
            sigG = S.sfft_signal_expsum(planG, w_d, a_d)
            outsG = tuple(torch.empty_like(o) for o in outs)
            for _ in range(args.warmup):
                S.sfft_execute(planG, sigG, outsG)
            msG, repsG = time_steps(S, planG, sigG, outsG, args.spec_steps, stream, flush, barrier)
            msG = max_over_ranks(msG)
            spec_b[f"G{G}"] = {"value": mult * T * cfg.k * args.spec_steps / (msG / 1e3), "unit": "modes/s",
                               "ms_per_step": msG / args.spec_steps, "iterations": max(r.iterations for r in repsG),
                               "samples_per_step": sum(r.samples_used for r in repsG) / args.spec_steps,
                               "verified_exact_recovery": exact(outsG)}
            del planG, sigG, outsG

    # e2e: the public host-buffer calls, H2D of every step's inputs and D2H of its result inside the timed region.
    # (1) sfft_solve_host_batches: the K steps' batches in one call, the library overlapping each step's transfers
    # with its neighbours' solves (the headline e2e); (2) sfft_solve_host once per step (copies serialised with the
    # solve, L2 flushed between steps), reported alongside
    ne = args.steps if args.e2e_steps < 0 else args.e2e_steps
    e2e_value = e2e_serial = None
    hout = (torch.empty((T, cfg.k, cfg.d), dtype=torch.int32).pin_memory(),
            torch.empty((T, cfg.k, 2), dtype=torch.float64).pin_memory(),
            torch.empty((T,), dtype=torch.int32).pin_memory(),
            torch.empty((T,), dtype=torch.int32).pin_memory())
    h2d = w_h.numel() * 4 + a_h.numel() * 16
    d2h = hout[0].numel() * 4 + hout[1].numel() * 8 + hout[2].numel() * 4 + hout[3].numel() * 4
    if ne:
        wb = w_h.unsqueeze(0).expand(ne, *w_h.shape).contiguous().pin_memory()   # a copy per step (no reuse)
        ab = a_h.unsqueeze(0).expand(ne, *a_h.shape).contiguous().pin_memory()
        bout = (torch.empty((ne, T, cfg.k, cfg.d), dtype=torch.int32).pin_memory(),
                torch.empty((ne, T, cfg.k, 2), dtype=torch.float64).pin_memory(),
                torch.empty((ne, T), dtype=torch.int32).pin_memory(),
                torch.empty((ne, T), dtype=torch.int32).pin_memory())
        S.sfft_solve_host_batches(plan, wb, ab, bout)   # warm-up (allocates the second set and the streams; the
        # first DMA of fresh pinned pages is slow: C2's first call ran 1.06 vs 0.77 ms per step, tools/e2e_probe.py)
        # the consumer reads the warm-up's results (exact-recovery check) and the timed call must rewrite the counts
        # and statuses (sentinels; a CPU-written -1 over the whole freqs array would slow the DMA writes into those
        # lines: C2 0.91 vs 0.77 ms per step, tools/e2e_probe2.py)
        ok = ok and all(np.array_equal(bout[0][i].numpy(), ws) for i in range(ne))
        bout[2].fill_(-1)
        bout[3].fill_(-1)
        barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        S.sfft_solve_host_batches(plan, wb, ab, bout)
        e_ms = max_over_ranks((time.perf_counter() - t) * 1e3)
        for _ in range(int(os.environ.get("BENCH_E2E_DEBUG", "0"))):   # debugging aid: repeated calls on stderr
            t = time.perf_counter()
            S.sfft_solve_host_batches(plan, wb, ab, bout)
            print(f"[bench] e2e batches call {(time.perf_counter() - t) * 1e3 / ne:.3f} ms/step (first {e_ms / ne:.3f})",
                  file=sys.stderr)
        e2e_value = mult * T * cfg.k * ne / (e_ms / 1e3)
        ok = ok and all(np.array_equal(bout[0][i].numpy(), ws) for i in range(ne))
        ok = ok and bool((bout[2] == cfg.k).all()) and bool((bout[3] == 0).all())
        del wb, ab, bout
        S.sfft_solve_host(plan, w_h, a_h, hout)
        barrier()
        torch.cuda.synchronize()
        e_ms = 0.0
        for _ in range(ne):
            flush.zero_()
            torch.cuda.synchronize()
            t = time.perf_counter()
            S.sfft_solve_host(plan, w_h, a_h, hout)
            e_ms += (time.perf_counter() - t) * 1e3
        e_ms = max_over_ranks(e_ms)
        e2e_serial = mult * T * cfg.k * ne / (e_ms / 1e3)
        ok = ok and np.array_equal(hout[0].numpy(), ws)
    ok_t = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
    if world > 1:
        dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
    ok = bool(ok_t.item())

    # single-solve latency: one signal per execute (trial 0 of this rank), device-resident inputs,
    # CUDA events around each execute, median of the timed runs (not part of `value`)
    lat = None
    if args.latency_steps and not lines:
        plan1 = make_plan(args.expsum_path, batch=1, profile=False, shard=False)
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
        del plan1, sig1
        # multi-prime speculation (DESIGN reading R26, sfft_options.spec_primes = G): G primes per iteration in G
        # slots of one plan, merged in prime order -- fewer iterations for the same signal
        lat["speculation"] = {}
        for G in args.spec_primes:
            planG = S.sfft_plan(cfg.d, cfg.N, cfg.k, blocks=cfg.blocks, batch=1, expsum_path=args.expsum_path,
                                spec_primes=G)
            sigG = S.sfft_signal_expsum(planG, w_d[:1].contiguous(), a_d[:1].contiguous())
            for _ in range(2):
                S.sfft_execute(planG, sigG, outs1)
            tg = []
            for _ in range(args.latency_steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rg = S.sfft_execute(planG, sigG, outs1)
                e1.record(stream)
                torch.cuda.synchronize()
                tg.append(e0.elapsed_time(e1))
            lat["speculation"][f"G{G}"] = {"ms_median": sorted(tg)[len(tg) // 2], "iterations": rg.report.iterations,
                                           "samples": rg.report.samples_used,
                                           "exact": bool(np.array_equal(outs1[0][0].cpu().numpy(), ws[0]))}
            del planG, sigG

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = args.cpu_threads or os.cpu_count() or 1
        cpu, _ = oracle_run(cfg, cores, cores)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "modes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if lines else "weak",
            "vs_baseline": None,
            "dtype": f"int8-limb S={limbs} exp-sum + f64" if n8 else "f64",
            "dtype_note": ("exp-sum as exact int8 x int8 -> int32 limb products on tcgen05 combined in FP64 (reading "
                           "R22); FFT, decode, registry in FP64 / int64" if n8 else "FP64 / int64 throughout"),
            "data": "synthetic (seeded PCG64 per PAPER.md:424 recipe; no dataset exists for this metric)",
            "expsum_path": ("int8 limbs on tcgen05" if n8 else
                            "fp64, fused into the FFT CTAs" if tot("n_fused_sample") else "fp64"),
            "config": {"workload": workload_desc(cfg),
                       "signals_per_gpu_per_step": T,
                       "table_cache_slots": args.table_cache or f"plan default max(batch + 16, 512) = {max(T + 16, 512)}",
                       "parallelism": (f"prime-speculation ranks x{world} (one prime of each iteration per rank, NCCL "
                                       "record all-gather, merge in rank order)" if spec else
                                       f"line shards x{world} (" + ("records stored into every shard's memory by the FFT "
                                       "epilogue, CUDA IPC peer mappings" if args.exchange == "fused" else
                                       "NCCL record all-gather") + ")") if lines else f"signal shards x{world}",
                       "l2": "256 MB L2 flush between timed steps; per-step working set > 1 GB"},
            "sample_evals_per_s": mult * samples / (ms_max / 1e3),
            "verified_exact_recovery": ok,
            "roofline": roofline,
            "fft_roofline": fft_roof,
            "fp64_path": fp64,
            "speculation_batched": spec_b,
            "kernel_ms_per_step": {"expsum": ms_exp / args.steps, "fft": ms_fft / args.steps,
                                   "decode": ms_dec / args.steps, "other": ms_oth / args.steps,
                                   "profiled_step": ms_prof / args.steps,
                                   "note": "per-kernel-class CUDA events of a profiled plan (same signals, same steps); "
                                           "ms_per_step / value come from an unprofiled plan"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "modes/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": ne, "api": "sfft_solve_host_batches (pinned host buffers, one batch per step, transfers "
                                        "overlapped with the neighbouring steps' solves; wall clock; the previous "
                                        "call's results read on the host first, counts / statuses reset to -1)",
                    "serial_value": e2e_serial,
                    "serial_api": "sfft_solve_host once per step (H2D, solve, D2H in sequence, L2 flushed between "
                                  "steps; wall clock)"},
            "gpu_launches": launches,
            "latency_single_solve": lat,
            "clocks": clock_res,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: single-scan min-sum LDPC decoding on B200 (one process per GPU).

Headline workload (N=1): BASELINE.json configs[1] = config 2 (QC 35x59, Z=127, DTMB
shape, int16 Q3 LLRs at 1.5 dB, offset min-sum, <= 15 iterations with per-frame early
stop, 8192 frames per GPU); `--config k` selects another of the five BASELINE configs as
the headline.  A "step" is one ldpc_decode_batch of the whole per-GPU batch (all
iterations, syndrome checks, outputs) on inputs already in HBM.  The same run also times
all five configs (`per_config`, each with its own roofline, e2e and clocks), the GPU
two-scan / layered / §4 full-message forms of the headline workload, and the CPU oracle
(`cpu_baseline`).

Multi-GPU: `--gpus N` (N > 1) without a launcher re-executes itself under
torch.distributed.run (NCCL_DEBUG=INFO); under torchrun each rank decodes its own frame
shard (global frames [r*F, (r+1)*F)), weak scaling, all times are the max over ranks and
the error counters are all-reduced over NCCL after the timed region.  `--dist-check`
runs the same multi-rank plumbing (spawn, rendezvous, sharding, SUM/MAX all-reduce)
without decoding, on NCCL or, without GPUs, gloo.  `--impl reference` times the CPU
oracle (the paper's method as plain C) instead.

Prints ONE JSON line (rank 0).
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ldpcgen as g  # noqa: E402

METRIC = "decoded info Gbit/s and edge-updates/s at 1/2/4/8 B200; % HBM roofline"
UNIT = "Gbit/s"
L2_FLUSH_BYTES = 256 << 20
HEADLINE = 2          # BASELINE.json configs[1] (the task's default workload at N=1)

# Algorithmic bytes per edge-update (PAPER.md P:331-335 persistent-data model: read
# Z^(k-1) and Z^(0), write Z^(k), read+write the compact state per check, and for the
# 1-bit format read+write the per-edge sign bit): SURVEY.md §8(d)
#   bytes/iter/frame = N (w_Z0 + 2 w_L) + 2 M w_state + 2 E w_edge
W_BYTES = {1: (2, 2, 4, 0), 2: (2, 2, 4, 0), 3: (1, 2, 2.375, 1 / 8), 4: (2, 2, 4, 0), 5: (4, 4, 12, 0)}
# Algorithmic integer operations per edge-update of the method:
# rebuild L_old = s f(A,B,n,ñ) (compare n==ñ, select, sign: 3), q = Z - L_old (1),
# |q| and sgn q (2), two-minimum update (compare + 2 selects: 3), sign product (1),
# new message (compare, select, sign of the others, apply: 4), Z += L (1) = 15.
ALG_OPS_PER_EU = 15
# integer-pipe peaks per SM per clock (thread-instructions): the ALU pipe alone (unit count,
# B300_MICROARCH.md; confirmed 64.0 by tools/alu_peak.cu) and the measured LOP3 + IMAD
# dual-issue rate (profiles/r01_alu_peak.json), the ceiling once work is spread over the
# ALU and FMA pipes
ALU_PIPE_PER_CLK = 64.0
ALU_DUAL_PER_CLK = 86.4
GRAPH_DECODES = 64    # cfg1: one timed sample = a CUDA graph of 64 decodes of distinct batches


def describe(cfg, code):
    kinds = {g.LLR_I16: "int16 Q3", g.LLR_I8: "int8 Q2", g.LLR_F32: "fp32"}
    var = (f"offset {cfg.offset_raw} LSB" if cfg.variant == "offset" else f"normalized alpha={cfg.alpha}")
    stop = "early stop" if cfg.early_stop else "fixed"
    return (f"cfg{cfg.idx}: {cfg.code_kind} N={code.n_vars} M={code.n_checks} E={code.n_edges}, {kinds[cfg.llr_kind]} "
            f"LLRs at {cfg.ebn0_db} dB, {var}, {cfg.max_iter} it {stop}, {cfg.msg_format} messages, "
            f"{cfg.frames} frames/GPU")


def bytes_per_eu(cfg, code):
    wz, wl, ws, we = W_BYTES[cfg.idx]
    return (code.n_vars * (wz + 2 * wl) + 2 * code.n_checks * ws + 2 * code.n_edges * we) / code.n_edges


def dtype_name(cfg):
    """The arithmetic type of the path: 16-bit integer lanes (two frames per 32-bit register,
    int8 inputs widened on load) or fp32 messages (posterior sums exact in int64, D28)."""
    return "f32" if cfg.llr_kind == g.LLR_F32 else "int16"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during a timed region."""

    def __init__(self, device_index, tag=""):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_dev{device_index}{tag}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.2)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[4 + i] and "Not" not in r[4 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU oracle
def cpu_oracle_throughput(cfg, code, engine, budget_s, nthreads=0, start_frames=16):
    """Time the oracle as it stands on the host's cores over a bounded sample of the
    workload (frames from the same generator); returns (info Gbit/s, EU/s, frames, threads, seconds)."""
    import oracle
    mode = "f32" if cfg.llr_kind == g.LLR_F32 else "int"
    nt = nthreads or oracle.hardware_threads()
    F = max(start_frames, nt)
    while True:
        llr = cfg.llrs(code, 0, F)
        z = llr if mode == "f32" else llr.astype(np.int32)
        t0 = time.perf_counter()
        r = oracle.decode(code, z, engine, mode, cfg.max_iter, cfg.early_stop, cfg.offset_raw if mode == "int" else 0,
                          cfg.clamp if mode == "int" else 0, cfg.alpha, nthreads=nt)
        dt = time.perf_counter() - t0
        if dt >= budget_s * 0.5 or F >= 32768:
            eu = float(r.iters.sum()) * code.n_edges
            return F * code.K / dt / 1e9, eu / dt, F, r.threads, dt
        F = int(min(32768, F * max(2.0, budget_s * 0.8 / max(dt, 1e-3))))


def run_reference(args, cfg, code, rank, world):
    """--impl reference: the CPU oracle (compact single-scan, the paper's method) timed on
    host cores; under torchrun only rank 0 runs and prints."""
    if rank != 0:
        return
    import oracle
    nt = oracle.hardware_threads()
    if args.ref_frames:
        F = args.ref_frames
    else:
        budget = max(1.0, 120.0 / max(1, args.steps + args.warmup))
        _, _, F, _, _ = cpu_oracle_throughput(cfg, code, "compact", min(budget, 5.0), nt)
    llr = cfg.llrs(code, 0, F)
    mode = "f32" if cfg.llr_kind == g.LLR_F32 else "int"
    z = llr if mode == "f32" else llr.astype(np.int32)
    times, eus = [], []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = oracle.decode(code, z, "compact", mode, cfg.max_iter, cfg.early_stop, cfg.offset_raw if mode == "int" else 0,
                          cfg.clamp if mode == "int" else 0, cfg.alpha, nthreads=nt)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            eus.append(float(r.iters.sum()) * code.n_edges)
    tot = sum(times)
    value = args.steps * F * code.K / tot / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32" if mode == "int" else "f32",
            "data": "synthetic", "edge_updates_per_s": sum(eus) / tot,
            "config": {"workload": describe(cfg, code), "frames_per_step": F, "engine": "oracle compact single-scan"},
            "cpu_baseline": {"kind": "oracle", "value": value, "unit": UNIT, "cores": nt, "cpu_model": cpu_model(),
                             "sample": f"{F} frames of the workload per step, all host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- multi-rank
def spawn_ranks(argv, n):
    """Re-execute this script under torch.distributed.run with n ranks (one per GPU)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd, env=env)


def init_dist(world, local, use_cuda):
    import torch
    import torch.distributed as dist
    if world <= 1:
        return None
    os.environ.setdefault("NCCL_DEBUG", "INFO")        # the NCCL ranks / transports go on record
    if use_cuda:
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    return dist


def run_dist_check(args, cfg, code, rank, world, local):
    """The multi-rank plumbing of the bench without decoding: each rank takes its frame
    shard, counts the raw hard-decision errors of its channel LLRs (x^ = [LLR <= 0]), and
    the SUM / MAX all-reduce is checked on rank 0 against the single-process count of all
    frames.  NCCL when CUDA is available, else gloo (CPU)."""
    import torch
    import torch.distributed as tdist
    from paper_cs_0609090_b200.dist import frame_shard, reduce_counters
    use_cuda = torch.cuda.is_available()
    dev = torch.device("cuda", local) if use_cuda else torch.device("cpu")
    if use_cuda:
        torch.cuda.set_device(local)
    # the process group is created even for one rank, so the NCCL init and all-reduce run on
    # a single-GPU box too
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if "MASTER_PORT" not in os.environ:
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
        sk.close()
    if use_cuda:
        tdist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    else:
        tdist.init_process_group("gloo", rank=rank, world_size=world)
    dist = tdist
    F = args.frames or 16

    def counts(f0, nf):
        llr = cfg.llrs(code, f0, nf)
        bad = (llr <= 0).sum(axis=1).astype(np.int64)
        return [int(bad.sum()), int((bad > 0).sum()), 0, int((bad > 0).sum()), 0]

    f0, nf = frame_shard(rank, world, F)
    c = torch.tensor(counts(f0, nf), dtype=torch.int64, device=dev)
    t = torch.tensor([1.0 + rank], dtype=torch.float64, device=dev)
    if world > 1:
        reduce_counters(c, t)
    else:                                              # reduce_counters skips one rank; run the collectives anyway
        tdist.all_reduce(c, op=tdist.ReduceOp.SUM)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    if rank == 0:
        want = counts(0, F * world)
        got = c.cpu().tolist()
        line = {"dist_check": got == want and float(t.item()) == float(world), "n_ranks": world,
                "backend": tdist.get_backend(), "counters": got, "expected": want,
                "max_elapsed": float(t.item()), "frames_per_rank": F}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


# ----------------------------------------------------------------------------- GPU timing
class Ctx:
    """Per-rank state shared by the measurements."""

    def __init__(self, args, rank, world, local, dist):
        import torch
        self.torch = torch
        self.args, self.rank, self.world, self.local, self.dist = args, rank, world, local, dist
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream(self.dev)
        self.flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=self.dev)
        self.peaks, self.peak_src = load_peaks()

    def max_over_ranks(self, x):
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def time_calls(self, fn, n, flush=True):
        """n calls of fn, each bracketed by CUDA events on this rank's stream (L2 flushed
        before each, outside the events); returns the per-call times in ms."""
        torch = self.torch
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        self.barrier()
        torch.cuda.synchronize(self.dev)
        for i in range(n):
            if flush:
                self.flush.fill_(i & 0xFF)
            evs[i][0].record(self.stream)
            fn()
            evs[i][1].record(self.stream)
        torch.cuda.synchronize(self.dev)
        self.barrier()
        return [a.elapsed_time(b) for a, b in evs]


def measure_config(ctx, cfg, steps, warmup, want_e2e=True):
    """Time one BASELINE config on this rank's frame shard: the device-resident decode
    (value), its roofline, the end-to-end host-buffer decode (e2e) and the clocks.  All times
    are the max over ranks."""
    import paper_cs_0609090_b200 as P
    from paper_cs_0609090_b200.dist import frame_shard, reduce_counters
    torch = ctx.torch
    code = cfg.code()
    f0, F = frame_shard(ctx.rank, ctx.world, cfg.frames)
    llr_host = cfg.llrs(code, f0, F)
    llr = torch.from_numpy(llr_host).to(ctx.dev)
    dec = P.Decoder(code, ctx.local)
    params = P.params_for_config(cfg)
    out = dec.alloc_outputs(F, params.llr_type, posteriors=True)
    for _ in range(warmup):
        dec.decode(llr, params, out)
    torch.cuda.synchronize(ctx.dev)
    launches = P.ldpc_last_launch_count()
    graph = None
    if cfg.idx == 1:
        # a decode is ~0.1 ms, so one timed sample is a CUDA graph of GRAPH_DECODES
        # decodes, of distinct batches whose inputs together exceed the L2 (no flush inside)
        nb = GRAPH_DECODES
        batches = [torch.from_numpy(cfg.llrs(code, f0 + 1_000_000 * (b + 1), F)).to(ctx.dev) for b in range(nb)]
        outs = [dec.alloc_outputs(F, params.llr_type, posteriors=True) for _ in range(nb)]
        s = torch.cuda.Stream(ctx.dev)
        s.wait_stream(ctx.stream)
        with torch.cuda.stream(s):
            for b in range(nb):            # warm the capture stream (no first-call work inside the capture)
                dec.decode(batches[b], params, outs[b])
        torch.cuda.synchronize(ctx.dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for b in range(nb):
                dec.decode(batches[b], params, outs[b])
        graph.replay()
        torch.cuda.synchronize(ctx.dev)
    sampler = ClockSampler(ctx.local, f"_cfg{cfg.idx}")
    sampler.start()
    if graph is not None:
        samples = ctx.time_calls(graph.replay, steps)
        step_ms = [t / GRAPH_DECODES for t in samples]
        decodes = steps * GRAPH_DECODES
    else:
        step_ms = ctx.time_calls(lambda: dec.decode(llr, params, out), steps)
        decodes = steps
    clocks = sampler.stop()
    ms = ctx.max_over_ranks(statistics.mean(step_ms))
    counters = dec.count_errors(out)
    reduce_counters(counters, torch.zeros(1, dtype=torch.float64, device=ctx.dev))
    c = counters.cpu().numpy().tolist()
    my_eu = float(out.iterations.sum().item()) * code.n_edges
    eu_step = float(c[4]) * code.n_edges                           # all ranks
    info_bits = float(ctx.world) * F * code.K
    value = info_bits / (ms * 1e-3) / 1e9
    eu_s = eu_step / (ms * 1e-3)
    bpe = bytes_per_eu(cfg, code)
    my_ms = statistics.mean(step_ms)
    hbm_model = {"bytes_per_eu": bpe, "achieved_gbs": bpe * my_eu / (my_ms * 1e-3) / 1e9,
                 "peak_gbs": ctx.peaks["hbm_gbs"], "peak_source": ctx.peak_src}
    hbm_model["frac"] = hbm_model["achieved_gbs"] / ctx.peaks["hbm_gbs"]
    hbm_model["frac_of_nominal_8tbs"] = hbm_model["achieved_gbs"] / 8000.0
    resident = launches == 1
    if resident:
        clk = (clocks or {}).get("sm_mhz") or ctx.peaks.get("sm_max_mhz", 1965.0)
        achieved = ALG_OPS_PER_EU * my_eu / (my_ms * 1e-3) / 1e12
        peak_pipe = 148 * ALU_PIPE_PER_CLK * 2 * clk * 1e6 / 1e12
        peak_dual = 148 * ALU_DUAL_PER_CLK * 2 * clk * 1e6 / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_pipe, "unit": "Tops/s", "frac": achieved / peak_pipe,
                "traffic": None, "peak_source": "derived: 148 SMs x 64 thread-instr/clk/SM (ALU pipe) x 2 frames per "
                                                "16x2 lane x SM clock under load (DESIGN.md §5.2)",
                "peak_dual_issue": peak_dual, "frac_dual_issue": achieved / peak_dual,
                "how": (f"{ALG_OPS_PER_EU} algorithmic 16-bit ops per edge-update x edge-updates of the launch / its "
                        f"duration (the decode is one launch); dual-issue peak: the measured LOP3+IMAD rate "
                        f"{ALU_DUAL_PER_CLK}/clk/SM (profiles/r01_alu_peak.json)"),
                "hbm_model": hbm_model}
    else:
        # Streaming: one iteration-kernel launch per iteration plus a few per-decode launches
        # (ingest, final syndrome, outputs).  The iteration kernel's average launch duration
        # is measured live as the slope of the step time over max_iter (the same frames
        # decoded with max_iter and max_iter - D, timed on this stream like the steps).
        it_ms = None
        if not cfg.early_stop and cfg.max_iter > 10:
            D = cfg.max_iter // 2
            short = P.params_for_config(cfg)
            short.max_iter = cfg.max_iter - D
            so = dec.alloc_outputs(F, short.llr_type, posteriors=True)
            dec.decode(llr, short, so)
            t_short = ctx.time_calls(lambda: dec.decode(llr, short, so), max(3, min(steps, 5)))
            it_ms = (my_ms - statistics.mean(t_short)) / D
            del so
        eu_iter = my_eu / cfg.max_iter
        if it_ms and it_ms > 0:
            ach = bpe * eu_iter / (it_ms * 1e-3) / 1e9
            how = (f"iteration-kernel launch: (step time at max_iter - at max_iter-{cfg.max_iter // 2}) / "
                   f"{cfg.max_iter // 2} = {it_ms:.4f} ms per launch, algorithmic bytes per launch "
                   f"{bpe * eu_iter / 1e6:.1f} MB")
        else:
            ach = hbm_model["achieved_gbs"]
            how = "algorithmic bytes of the whole step / step time (lower bound of the iteration kernel's rate)"
        roof = {"bound": "hbm", "achieved": ach, "peak": ctx.peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / ctx.peaks["hbm_gbs"], "traffic": None, "peak_source": ctx.peak_src,
                "frac_of_nominal_8tbs": ach / 8000.0, "how": how, "kernel_ms_per_launch": it_ms,
                "whole_step": hbm_model}
        if it_ms and it_ms > 0 and cfg.llr_kind != g.LLR_F32:
            # the integer streaming kernel issues the same 16x2 row arithmetic as the resident
            # one; ncu shows it issue/ALU-limited as much as byte-limited, so
            # the ALU-pipe fraction is reported beside the HBM one
            clk = (clocks or {}).get("sm_mhz") or ctx.peaks.get("sm_max_mhz", 1965.0)
            a_ach = ALG_OPS_PER_EU * eu_iter / (it_ms * 1e-3) / 1e12
            a_peak = 148 * ALU_PIPE_PER_CLK * 2 * clk * 1e6 / 1e12
            roof["alu_model"] = {"achieved": a_ach, "peak": a_peak, "unit": "Tops/s", "frac": a_ach / a_peak,
                                 "how": f"{ALG_OPS_PER_EU} algorithmic 16-bit ops per edge-update, iteration-kernel "
                                        f"launch duration; peak as the resident kernels' (DESIGN.md §5.2)"}
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{cfg.idx}.json")   # tools/ncu_summary.py
    if os.path.exists(prof):
        with open(prof) as f:
            pj = json.load(f)
        fp = pj.get("frames_profiled") or F
        roof["traffic"] = pj.get("dram_bytes_per_launch") * F / fp      # per launch of this run's batch
        roof["traffic_source"] = (pj.get("source", os.path.relpath(prof, ROOT)) +
                                  (f", scaled from {fp} to {F} frames" if fp != F else ""))
    res = {"value": value, "unit": UNIT, "ms_per_step": ms, "edge_updates_per_s": eu_s, "dtype": dtype_name(cfg),
           "workload": describe(cfg, code), "frames_per_gpu": F, "info_bits_per_frame": code.K,
           "mean_iterations": c[4] / (F * ctx.world), "frames_converged": ctx.world * F - c[3],
           "errors": {"bit_errors": c[0], "frame_errors": c[1], "undetected": c[2], "not_converged": c[3]},
           "roofline": roof, "clocks": clocks, "gpu_launches_per_step": launches,
           "timing": (f"CUDA graph of {GRAPH_DECODES} decodes of distinct batches per sample (inputs exceed L2), "
                      f"{steps} samples" if graph is not None else
                      f"{steps} steps, L2 flushed between steps (256 MiB write)"),
           "decodes_timed": decodes, "code_sha256": code.sha256()[:16]}
    if want_e2e:
        res["e2e"] = measure_e2e(ctx, dec, params, llr_host, F, code, info_bits, steps)
    res["_dec"], res["_llr"], res["_code"], res["_F"], res["_info_bits"] = dec, llr, code, F, info_bits
    return res


def measure_e2e(ctx, dec, params, llr_host, F, code, info_bits, steps):
    """The same metric through the C ABI's host-buffer entry point: H2D of the LLRs and
    D2H of hard bits, posteriors, flags and iteration counts inside the timed region."""
    torch = ctx.torch
    lh = torch.from_numpy(llr_host).pin_memory()
    hbh = torch.empty((F, dec.wpf), dtype=torch.int32).pin_memory()
    okh = torch.empty(F, dtype=torch.uint8).pin_memory()
    ith = torch.empty(F, dtype=torch.int32).pin_memory()
    post_dt = torch.float32 if llr_host.dtype == np.float32 else torch.int16
    ph = torch.empty((F, code.n_vars), dtype=post_dt).pin_memory()
    for _ in range(2):
        dec.decode_host(lh, params, hbh, okh, ith, ph)
    torch.cuda.synchronize(ctx.dev)
    e_ms = ctx.time_calls(lambda: dec.decode_host(lh, params, hbh, okh, ith, ph), max(3, min(steps, 10)))
    ms = ctx.max_over_ranks(statistics.mean(e_ms))
    return {"value": info_bits / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": int(llr_host.nbytes),
            "d2h_bytes_per_step": int(hbh.numel() * 4 + okh.numel() + ith.numel() * 4 + ph.numel() * ph.element_size()),
            "api": "ldpc_decode_batch_host (pinned host buffers; copies overlap decoding in frame chunks)"}


def time_schedule(ctx, cfg, res, sched, msg_format=None, steps=5):
    """The headline frames through another schedule / message format, timed the same way:
    the paper's comparison against two-scan, the layered schedule
    (§8(f2)) and the §4 per-edge form."""
    import paper_cs_0609090_b200 as P
    dec, llr, code, F = res["_dec"], res["_llr"], res["_code"], res["_F"]
    sp = P.params_for_config(cfg, sched, msg_format)
    try:
        dec.workspace(F, sp)
    except P.LdpcError as ex:
        return {"unsupported": str(ex)}
    so = dec.alloc_outputs(F, sp.llr_type, posteriors=True)
    dec.decode(llr, sp, so)
    t = ctx.time_calls(lambda: dec.decode(llr, sp, so), max(2, min(steps, 5)))
    ms = ctx.max_over_ranks(statistics.mean(t))
    v = res["_info_bits"] / (ms * 1e-3) / 1e9
    its = float(so.iterations.double().mean().item())
    return {"value": v, "unit": UNIT, "ms_per_step": ms,
            "edge_updates_per_s": its * F * ctx.world * code.n_edges / (ms * 1e-3),
            "mean_iterations": its, "frames_converged": int(so.syndrome_ok.sum().item()),
            "singlescan_over_this": res["value"] / v if v else None}


def strip(d):
    return {k: v for k, v in d.items() if not k.startswith("_")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=HEADLINE, choices=[1, 2, 3, 4, 5], help="headline config")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=0, help="override frames per GPU (headline config)")
    ap.add_argument("--ref-frames", type=int, default=0, help="--impl reference: frames per step (0 = sized by budget)")
    ap.add_argument("--dist-check", action="store_true", help="multi-rank plumbing check without decoding")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-twoscan", action="store_true", help="skip timing the GPU two-scan baseline")
    ap.add_argument("--no-layered", action="store_true", help="skip timing the layered / full-message forms")
    ap.add_argument("--no-per-config", action="store_true", help="skip timing the other four configs")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(sys.argv[1:], args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    cfg = g.CONFIGS[args.config]
    if args.frames:
        cfg.frames = args.frames
    code = cfg.code()

    if args.impl == "reference":
        return run_reference(args, cfg, code, rank, world)
    if args.dist_check:
        return run_dist_check(args, cfg, code, rank, world, local)

    import torch
    torch.cuda.set_device(local)
    dist = init_dist(world, local, True)
    ctx = Ctx(args, rank, world, local, dist)

    res = measure_config(ctx, cfg, args.steps, args.warmup, want_e2e=not args.no_e2e)
    twoscan = layered = fullmsg = None
    import paper_cs_0609090_b200 as P
    if not args.no_twoscan:
        twoscan = time_schedule(ctx, cfg, res, P.LDPC_SCHED_TWOSCAN)
        twoscan["paper_claim"] = "single-scan more than twice as fast as two-scan min-sum (PAPER.md P:29-30)"
    if not args.no_layered:
        layered = time_schedule(ctx, cfg, res, P.LDPC_SCHED_LAYERED)
        fullmsg = time_schedule(ctx, cfg, res, P.LDPC_SCHED_SINGLESCAN, P.LDPC_MSG_FULL)
    per_config = None
    if not args.no_per_config:
        per_config = {}
        for k in (1, 2, 3, 4, 5):
            if k == args.config:
                per_config[f"cfg{k}"] = "headline (this line)"
                continue
            r = measure_config(ctx, g.CONFIGS[k], min(args.steps, 5), 3, want_e2e=not args.no_e2e)
            per_config[f"cfg{k}"] = strip(r)
            del r
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gb, eus, Fs, nt, dt = cpu_oracle_throughput(cfg, code, "compact", args.cpu_budget)
        gb2, eus2, Fs2, nt2, dt2 = cpu_oracle_throughput(cfg, code, "twoscan", args.cpu_budget / 2)
        g1, e1, F1, _, d1 = cpu_oracle_throughput(cfg, code, "compact", min(3.0, args.cpu_budget / 4), nthreads=1,
                                                   start_frames=1)
        cpu = {"value": gb, "unit": UNIT, "cores": nt, "kind": "oracle",
               "sample": f"{Fs} frames of the workload (compact single-scan oracle, {dt:.1f} s, all host threads)",
               "cpu_model": cpu_model(), "edge_updates_per_s": eus,
               "single_thread": {"value": g1, "edge_updates_per_s": e1, "frames": F1, "seconds": d1},
               "twoscan": {"value": gb2, "edge_updates_per_s": eus2, "frames": Fs2},
               "singlescan_over_twoscan": gb / gb2 if gb2 else None,
               "paper_claim": "single-scan min-sum more than twice as fast as two-scan (PAPER.md P:29-30)"}

    if rank == 0:
        launches = res["gpu_launches_per_step"]
        line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": res["dtype"], "data": "synthetic",
                "edge_updates_per_s": res["edge_updates_per_s"],
                "config": {"workload": res["workload"], "frames_per_gpu": res["frames_per_gpu"],
                           "global_frames": res["frames_per_gpu"] * world,
                           "parallelism": f"dp{world} (frames sharded, counters all-reduced over NCCL)",
                           "info_bits_per_frame": res["info_bits_per_frame"], "l2": res["timing"],
                           "code_sha256": res["code_sha256"]},
                "errors": dict(res["errors"], mean_iterations=res["mean_iterations"]),
                "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res.get("e2e"),
                "gpu_twoscan": twoscan, "gpu_layered": layered, "gpu_full_messages": fullmsg,
                "per_config": per_config,
                "gpu_launches": launches * res["decodes_timed"], "clocks": res["clocks"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

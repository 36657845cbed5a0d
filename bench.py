#!/usr/bin/env python
"""Benchmark: single-scan min-sum LDPC decoding on B200 (one process per GPU).

Default workload (N=1): BASELINE.json configs[1] = config 2 (QC 35x59, Z=127,
DTMB shape, int16 Q3 LLRs at 1.5 dB, offset min-sum, <= 15 iterations with
per-frame early stop, 8192 frames per GPU).  `--config k` selects another of the
five BASELINE configs.  A "step" is one ldpc_decode_batch of the whole per-GPU
batch (all iterations, syndrome checks, outputs) on inputs already in HBM.

Prints ONE JSON line (rank 0).  Under torchrun each rank decodes its own frame
shard (global frames [r*F, (r+1)*F)), weak scaling, and the bit/frame error
counters are all-reduced over NCCL after the timed region.
`--impl reference` times the CPU oracle (the paper's method as plain C) instead.
"""
import argparse
import json
import os
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

# Algorithmic bytes per edge-update (PAPER.md P:331-335 persistent-data model:
# read Z^(k-1) and Z^(0), write Z^(k), read+write the compact state per check):
# bytes/iter/frame = N (w_Z0 + 2 w_L) + 2 M w_state.
W_BYTES = {1: (2, 2, 4), 2: (2, 2, 4), 3: (1, 2, 2.375), 4: (2, 2, 4), 5: (4, 4, 12)}
# Algorithmic integer operations per edge-update of the method:
# rebuild L_old = s f(A,B,n,ñ) (compare n==ñ, select, sign: 3), q = Z - L_old (1),
# |q| and sgn q (2), two-minimum update (compare + 2 selects: 3), sign product (1),
# new message (compare, select, sign of the others, apply: 4), Z += L (1) = 15.
ALG_OPS_PER_EU = 15


def describe(cfg, code):
    kinds = {g.LLR_I16: "int16 Q3", g.LLR_I8: "int8 Q2", g.LLR_F32: "fp32"}
    var = (f"offset {cfg.offset_raw} LSB" if cfg.variant == "offset" else f"normalized alpha={cfg.alpha}")
    stop = "early stop" if cfg.early_stop else "fixed"
    return (f"cfg{cfg.idx}: {cfg.code_kind} N={code.n_vars} M={code.n_checks} E={code.n_edges}, {kinds[cfg.llr_kind]} "
            f"LLRs at {cfg.ebn0_db} dB, {var}, {cfg.max_iter} it {stop}, {cfg.msg_format} messages, "
            f"{cfg.frames} frames/GPU")


def bytes_per_eu(cfg, code):
    wz, wl, ws = W_BYTES[cfg.idx]
    return (code.n_vars * (wz + 2 * wl) + 2 * code.n_checks * ws) / code.n_edges


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_dev{device_index}.csv")

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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, cfg, code, rank, world):
    """--impl reference: the CPU oracle (compact single-scan, the paper's method) timed on host cores."""
    if rank != 0:
        return
    import oracle
    nt = oracle.hardware_threads()
    budget = max(1.0, 120.0 / max(1, args.steps + args.warmup))
    # size the per-step sample once
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=0, help="override frames per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-twoscan", action="store_true", help="skip timing the GPU two-scan baseline")
    ap.add_argument("--no-layered", action="store_true", help="skip timing the layered schedule")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = g.CONFIGS[args.config]
    if args.frames:
        cfg.frames = args.frames
    code = cfg.code()

    if args.impl == "reference":
        return run_reference(args, cfg, code, rank, world)

    import torch
    import torch.distributed as dist
    import paper_cs_0609090_b200 as P

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_cs_0609090_b200.dist import frame_shard, reduce_counters
    f0, F = frame_shard(rank, world, cfg.frames)
    llr_host = cfg.llrs(code, f0, F)                      # this rank's global frame shard
    llr = torch.from_numpy(llr_host).to(dev)
    dec = P.Decoder(code, local)
    params = P.params_for_config(cfg)
    out = dec.alloc_outputs(F, params.llr_type, posteriors=True)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        dec.decode(llr, params, out)
    torch.cuda.synchronize(dev)
    launches_per_step = P.ldpc_last_launch_count()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        flush.fill_(i & 0xFF)                             # L2 flush between steps (not timed)
        evs[i][0].record(stream)
        dec.decode(llr, params, out)
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)

    # iterations / error counters of the last step (all steps decode the same frames)
    counters = dec.count_errors(out)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    reduce_counters(counters, t)                          # NCCL: SUM counters, MAX elapsed
    total_ms = float(t.item())
    c = counters.cpu().numpy().tolist()
    sum_iters = c[4]
    eu_per_step = float(sum_iters) * code.n_edges               # all ranks
    info_bits_per_step = float(world) * F * code.K
    value = info_bits_per_step * args.steps / (total_ms * 1e-3) / 1e9
    eu_s = eu_per_step * args.steps / (total_ms * 1e-3)

    # ---- roofline of the dominant kernel (the decode is one resident launch, or the
    # per-iteration streaming launches): measured per-step on this rank's stream
    peaks, peak_src = load_peaks()
    my_eu = float(out.iterations.sum().item()) * code.n_edges
    my_ms = statistics.mean(step_ms)
    resident = launches_per_step == 1
    if resident:
        clk = (clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        # 16-bit integer ops: ALU pipe 64 lanes/clk/SM (VIADD/VIMNMX/LOP3/PRMT all issue
        # there) x 2 frames per lane (16x2 SIMD) x 148 SMs x SM clock
        peak_ops = 148 * 64 * 2 * clk * 1e6 / 1e12
        achieved = ALG_OPS_PER_EU * my_eu / (my_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_ops, "unit": "Tops/s",
                "frac": achieved / peak_ops, "traffic": None,
                "how": (f"{ALG_OPS_PER_EU} algorithmic 16-bit ops per edge-update x edge-updates of the "
                        f"launch / its duration (the decode is one launch); peak derived: 148 SMs x 64 "
                        f"thread-instr/clk/SM on the ALU pipe (confirmed by tools/alu_peak.cu, "
                        f"profiles/r01_alu_peak.json) x 2 frames per 16x2 lane x {clk:.0f} MHz"),
                "hbm_model": {"bytes_per_eu": bytes_per_eu(cfg, code),
                              "achieved_gbs": bytes_per_eu(cfg, code) * my_eu / (my_ms * 1e-3) / 1e9,
                              "peak_gbs": peaks["hbm_gbs"],
                              "frac": bytes_per_eu(cfg, code) * my_eu / (my_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                              "frac_of_nominal_8tbs": bytes_per_eu(cfg, code) * my_eu / (my_ms * 1e-3) / 8e12}}
    else:
        # Streaming path: one iteration-kernel launch per iteration plus a few per-decode
        # launches (ingest, final syndrome, outputs).  The iteration kernel's average launch
        # duration is measured live as the slope of the step time over max_iter: the same
        # frames decoded with max_iter and max_iter - D, timed on this stream like the steps.
        ach_step = bytes_per_eu(cfg, code) * my_eu / (my_ms * 1e-3) / 1e9
        it_ms = None
        if not cfg.early_stop and cfg.max_iter > 10:
            D = cfg.max_iter // 2
            short = P.params_for_config(cfg)
            short.max_iter = cfg.max_iter - D
            so = dec.alloc_outputs(F, short.llr_type, posteriors=True)
            dec.decode(llr, short, so)
            torch.cuda.synchronize(dev)
            t_short = []
            for i in range(max(3, min(args.steps, 8))):
                flush.fill_(i & 0xFF)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                dec.decode(llr, short, so)
                b_.record(stream)
                b_.synchronize()
                t_short.append(a_.elapsed_time(b_))
            it_ms = (my_ms - statistics.mean(t_short)) / D
            del so
        eu_iter = my_eu / cfg.max_iter
        if it_ms and it_ms > 0:
            ach = bytes_per_eu(cfg, code) * eu_iter / (it_ms * 1e-3) / 1e9
            how = (f"iteration-kernel launch: (step time at max_iter - step time at max_iter-{cfg.max_iter // 2}) / "
                   f"{cfg.max_iter // 2} = {it_ms:.4f} ms per launch, algorithmic bytes per launch "
                   f"{bytes_per_eu(cfg, code) * eu_iter / 1e6:.1f} MB")
        else:
            ach = ach_step
            how = "algorithmic bytes of the whole step / step time (lower bound of the iteration kernel's rate)"
        roof = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": None, "frac_of_nominal_8tbs": ach / 8000.0,
                "how": how, "whole_step": {"achieved_gbs": ach_step, "frac": ach_step / peaks["hbm_gbs"]},
                "kernel_ms_per_launch": it_ms}
    roof["peak_source"] = "derived (unit counts x clock, microbenchmark-confirmed)" if resident else peak_src
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{cfg.idx}.json")   # from tools/ncu_summary.py
    if os.path.exists(prof):
        with open(prof) as f:
            roof["traffic"] = json.load(f).get("dram_bytes_per_launch")

    # ---- end to end through the C ABI with host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        lh = torch.from_numpy(llr_host).pin_memory()
        hbh = torch.empty((F, dec.wpf), dtype=torch.int32).pin_memory()
        okh = torch.empty(F, dtype=torch.uint8).pin_memory()
        ith = torch.empty(F, dtype=torch.int32).pin_memory()
        for _ in range(2):
            dec.decode_host(lh, params, hbh, okh, ith)
        torch.cuda.synchronize(dev)
        e_ms = []
        for i in range(max(3, min(args.steps, 10))):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dec.decode_host(lh, params, hbh, okh, ith)
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        te = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": info_bits_per_step * len(e_ms) / (float(te.item()) * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(llr_host.nbytes),
               "d2h_bytes_per_step": int(hbh.numel() * 4 + okh.numel() + ith.numel() * 4),
               "ms_per_step": float(te.item()) / len(e_ms)}

    # ---- the other schedules on the same frames, timed the same way (events on this
    # stream, L2 flushed): the paper's comparison against two-scan (SURVEY
    # §8(f1)) and the layered schedule (§8(f2), resident-kernel codes only)
    def time_schedule(sched, msg_format=None):
        sp = P.params_for_config(cfg, sched, msg_format)
        try:
            dec.workspace(F, sp)
        except P.LdpcError as ex:
            return {"unsupported": str(ex)}
        so = dec.alloc_outputs(F, sp.llr_type, posteriors=True)
        dec.decode(llr, sp, so)
        torch.cuda.synchronize(dev)
        t_ms = []
        for i in range(max(2, min(args.steps, 5))):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dec.decode(llr, sp, so)
            b.record(stream)
            b.synchronize()
            t_ms.append(a.elapsed_time(b))
        tt = torch.tensor([sum(t_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        v = info_bits_per_step * len(t_ms) / (float(tt.item()) * 1e-3) / 1e9
        its = float(so.iterations.double().mean().item())
        return {"value": v, "unit": UNIT, "ms_per_step": float(tt.item()) / len(t_ms),
                "edge_updates_per_s": its * F * world * code.n_edges * len(t_ms) / (float(tt.item()) * 1e-3),
                "mean_iterations": its, "frames_converged": int(so.syndrome_ok.sum().item()),
                "singlescan_over_this": value / v if v else None}

    twoscan = layered = fullmsg = None
    if not args.no_twoscan:
        twoscan = time_schedule(P.LDPC_SCHED_TWOSCAN)
        twoscan["paper_claim"] = "single-scan more than twice as fast as two-scan min-sum (PAPER.md P:29-30)"
    if not args.no_layered:
        layered = time_schedule(P.LDPC_SCHED_LAYERED)
        # the §4 single-scan with stored per-edge messages (LDPC_MSG_FULL, resident codes)
        fullmsg = time_schedule(P.LDPC_SCHED_SINGLESCAN, P.LDPC_MSG_FULL)

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
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f32" if cfg.llr_kind == g.LLR_F32 else ("int16x2" if cfg.llr_kind == g.LLR_I16 else "int8->int16x2"),
                "data": "synthetic", "edge_updates_per_s": eu_s,
                "config": {"workload": describe(cfg, code), "frames_per_gpu": F, "global_frames": F * world,
                           "parallelism": f"dp{world} (frames sharded, counters all-reduced over NCCL)",
                           "info_bits_per_frame": code.K, "l2": "flushed between timed steps (256 MiB write)",
                           "code_sha256": code.sha256()[:16]},
                "errors": {"bit_errors": c[0], "frame_errors": c[1], "undetected": c[2], "not_converged": c[3],
                           "mean_iterations": sum_iters / (F * world)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_twoscan": twoscan, "gpu_layered": layered,
                "gpu_full_messages": fullmsg,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

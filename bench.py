#!/usr/bin/env python
"""Benchmark of the GAP-LA layer-assignment hot path (DP + backtrack + commit + Elmore) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

One step = one pass of the whole hot path over the whole synthetic design:
la_reset (restore the initial demand, a device copy) + every conflict-free batch (la_assign_batch =
K4/K5 DP + backtrack, la_commit_demand = K8 commit [+ NCCL reconcile when N > 1]) + la_eval_timing
(K6/K7 Elmore).  Inputs (forest, grid state) are resident in HBM and far larger than L2.  Forest
build and batching (la_load_nets) are setup, reported separately; the e2e number includes them.

Rank 0 prints ONE JSON line (see DESIGN.md §8 for every field).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "nets layer-assigned/sec (DP+Elmore+commit) at 1/2/4/8 B200; % HBM roofline"
DEFAULT_CONFIG = 5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, help="BASELINE.json config (1-based)")
    ap.add_argument("--n-nets", type=int, default=None, help="override the config's net count")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU work of the oracle sample")
    ap.add_argument("--batching", choices=["conflict-free", "paper"], default="conflict-free",
                    help="conflict-free batches (exact sequential semantics, default) or the paper's Alg. 1 "
                         "snapshot batches (NEXT #1/#2, synthetic criticality)")
    ap.add_argument("--max-batch", type=int, default=1 << 18, help="Alg. 1 GetBatches size cap (paper batching)")
    ap.add_argument("--no-pre", action="store_true", help="skip the NEXT #2 measurements (pre-timing, Alg. 1)")
    ap.add_argument("--ncu-pre", action="store_true", help="--ncu-pass: also run la_pre_timing in the profiled region")
    ap.add_argument("--ncu-pass", action="store_true",
                    help="setup + 1 warm step, then ONE step between cudaProfilerStart/Stop (for ncu)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc, self.th = device, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def host_info():
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = "unknown"
    return model, os.cpu_count()


def algorithmic_bytes(st, L, n_nets, via_cuts=None):
    """SURVEY §8(d) d.4 per-unit algorithmic bytes, with the instance's exact counts:
    K4/K5 (k_assign): tree 32/node + sinks 9/pin + wire state 4/(unit edge, legal layer)
                      + via state 4/(node, cut) + decisions 3/node + f_root 8/net
    K8 (k_commit):   8 per unit edge + 8 per via cut (int32 read-modify-write)
    K6/K7 (k_elmore): 19/node + 17/sink + 16/net"""
    N, P = st["n_nodes"], st["n_sinks"]
    assign = 32 * N + 9 * P + 4 * st["wire_state_words"] + 4 * st["via_state_words"] + 3 * N + 8 * n_nets
    commit = 8 * st["wirelength"] + 8 * (via_cuts or 0)
    elmore = 19 * N + 17 * P + 16 * n_nets
    return assign, commit, elmore


def ncu_summary(workload):
    """The committed ncu summary of the k_assign launches (profiles/ncu_k_assign_summary.json) if it
    matches the workload: dram bytes per launch, FP64-pipe activity, source files."""
    p = os.path.join(ROOT, "profiles", "ncu_k_assign_summary.json")
    try:
        with open(p) as f:
            j = json.load(f)
        if j.get("workload") == workload:
            return j
    except Exception:
        pass
    return {}


# ------------------------------------------------------------------ reference arm (the CPU oracle)
def run_reference(args, rank):
    if rank != 0:
        return
    from gen import synth
    from oracle import oracle
    d = synth.make_config(args.config, n_nets=args.n_nets)
    # size each step as a bounded prefix (priority order) of the workload: ~args.cpu_seconds / (W+K) s each
    probe = oracle.run(d, solution=False, grids=False, timing=False, batches=False, max_nets=min(20000, d.n_nets))
    rate = probe["nets_run"] / max(probe["elapsed_s"], 1e-9)
    per_step_s = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    sample = int(min(d.n_nets, max(1000, rate * per_step_s)))
    for _ in range(args.warmup):
        oracle.run(d, solution=False, grids=False, timing=False, batches=False, max_nets=sample)
    vals = []
    for _ in range(args.steps):
        r = oracle.run(d, solution=False, grids=False, timing=False, batches=False, max_nets=sample)
        vals.append(r["nets_run"] / r["elapsed_s"])
    v = statistics.median(vals)
    model, ncpu = host_info()
    desc = (f"first {sample} nets (priority order) of {d.name}, sequential fp64 oracle, 1 thread on {model} "
            f"({ncpu} host cores); timed region = DP+backtrack+commit+Elmore, tree build excluded")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "nets/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sample / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": d.name, "sample_nets": sample},
        "cpu_baseline": {"value": v, "unit": "nets/s", "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": v, "unit": "nets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)


def cpu_baseline(d, seconds):
    from oracle import oracle
    probe = oracle.run(d, solution=False, grids=False, timing=False, batches=False, max_nets=min(20000, d.n_nets))
    rate = probe["nets_run"] / max(probe["elapsed_s"], 1e-9)
    sample = int(min(d.n_nets, max(1000, rate * seconds)))
    r = oracle.run(d, solution=False, grids=False, timing=False, batches=False, max_nets=sample)
    model, ncpu = host_info()
    return {"value": r["nets_run"] / r["elapsed_s"], "unit": "nets/s", "cores": 1, "kind": "oracle",
            "sample": (f"first {sample} nets (priority order) of {d.name}: sequential fp64 oracle, 1 thread of "
                       f"{ncpu} ({model}); {r['elapsed_s']:.1f} s of DP+backtrack+commit+Elmore, tree build excluded")}


def cpu_baseline_mode2(d, seconds, rate1):
    """SURVEY §8(d) d.5 mode 2: the oracle with the nets of each conflict-free batch on every host
    core (OpenMP; bit-equal to mode 1, tests/test_oracle_modes.py), over a bounded prefix."""
    from oracle import oracle
    model, ncpu = host_info()
    threads = max(1, ncpu or 1)
    sample = int(min(d.n_nets, max(1000, rate1 * seconds * threads * 0.5)))
    r = oracle.run(d, solution=False, grids=False, timing=False, batches=False, max_nets=sample, threads=threads)
    return {"value": r["nets_run"] / r["elapsed_s"], "unit": "nets/s", "cores": threads, "kind": "oracle mode 2",
            "sample": (f"first {sample} nets (priority order) of {d.name}: fp64 oracle, the nets of each "
                       f"conflict-free batch on {threads} threads ({model}); {r['elapsed_s']:.1f} s of "
                       f"DP+backtrack+commit+Elmore, tree build excluded")}


def pre_assignment(args, A, d, la, crit, st, hbm):
    """SURVEY §8(f) NEXT #2, outside the step: the pre-assignment pi-model timing on the 2D trees
    (la_pre_timing, k_pre_timing) and Alg. 1 lines 3-10 (la_paper_batches), each timed W + K times
    with CUDA events on the library stream.  Algorithmic bytes:
      k_pre_timing: 30 per node (kid 16, len 4, sink0 4, height 2, nsink 2, nkid 1, edir 1)
                    + 24 per sink (cap, input index, delay out) + 24 per net (node range, id, cap out)
      Alg. 1 kernels: 24 per net (pin_ptr, seg_ptr, criticality, batch id out) + 8 per pin (slack)
                    + 16 per segment (x1 y1 x2 y2); the two radix passes are implementation traffic."""
    n_pins = int(d.pin_ptr[-1])
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            A.profiling(True)
            A.profile(reset=True)
        la.la_pre_timing(A.ctx, n_pins, d.n_nets)
    p1 = A.profile(reset=True)
    pt_ms = p1["pretime_ms"] / max(p1["pretime_launches"], 1)
    pt_bytes = 30 * st["n_nodes"] + 24 * st["n_sinks"] + 24 * d.n_nets
    nb_paper = None
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            A.profile(reset=True)
        _, nb_paper = la.la_paper_batches(A.ctx, d, crit, 0.7, 3, args.max_batch)
    p2 = A.profile(reset=True)
    A.profiling(False)
    calls = max(p2["order_calls"], 1)
    ok_ms, oc_ms = p2["order_kernel_ms"] / calls, p2["order_ms"] / calls
    or_bytes = 24 * d.n_nets + 8 * n_pins + 16 * int(d.seg_ptr[-1])
    return {"pre_timing": {"kernel": "k_pre_timing (pi-model Elmore on the 2D trees, per-direction r_avg/c_avg)",
                           "bound": "hbm", "ms": pt_ms, "alg_bytes": pt_bytes,
                           "achieved": pt_bytes / (pt_ms / 1e3) / 1e9 if pt_ms else None, "peak": hbm,
                           "unit": "GB/s", "frac": pt_bytes / (pt_ms / 1e3) / 1e9 / hbm if pt_ms else None},
            "paper_batches": {"kernels": "k_crit_max, k_order_keys, 2 x CUB radix SortPairs, scans, k_batch_*",
                              "bound": "hbm", "kernel_ms": ok_ms, "call_ms_with_h2d": oc_ms, "alg_bytes": or_bytes,
                              "achieved": or_bytes / (ok_ms / 1e3) / 1e9 if ok_ms else None, "peak": hbm,
                              "unit": "GB/s", "frac": or_bytes / (ok_ms / 1e3) / 1e9 / hbm if ok_ms else None,
                              "batches": nb_paper, "max_batch": args.max_batch}}


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    from gen import synth
    from paper_2507_13375_b200 import la

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    d = synth.make_config(args.config, n_nets=args.n_nets)
    def fresh_nccl_id():
        """A new ncclUniqueId from rank 0 for every communicator (an id is not reused)."""
        if world == 1:
            return None
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(la.la_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        return bytes(buf.cpu().numpy().tobytes())

    nid = fresh_nccl_id()
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    snap = None
    t_setup = time.perf_counter()
    A = la.LayerAssigner(d, device=local_rank, rank=rank, world=world, nccl_id=nid, stream=stream.cuda_stream)
    crit = synth.criticality(d) if (args.batching == "paper" or not args.no_pre) else None
    if args.batching == "paper":
        snap, _ = la.la_paper_batches(A.ctx, d, crit, 0.7, 3, args.max_batch)   # Alg. 1 l.3-10 on the GPU
    nb = A.load(snapshot_batches=snap)
    setup_s = time.perf_counter() - t_setup
    st0 = A.stats()

    def step():
        A.reset()
        A.assign_all()
        la.la_eval_timing(A.ctx)   # device outputs only; synchronises

    for _ in range(max(args.warmup, 1)):
        step()
    if args.ncu_pass:
        barrier()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        step()
        if args.ncu_pre:      # NEXT #2 kernels after the step (not part of it)
            la.la_pre_timing(A.ctx, int(d.pin_ptr[-1]), d.n_nets)
        torch.cuda.profiler.stop()
        if rank == 0:
            print(json.dumps({"ncu_pass": True, "workload": d.name, "batches": nb}), flush=True)
        return

    A.profiling(True)
    A.profile(reset=True)
    launches0 = A.stats()["launches"]
    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    prof = A.profile(reset=True)
    A.profiling(False)
    launches = (A.stats()["launches"] - launches0) // args.steps   # library kernels per timed step
    # evaluator (outside the step): Eq. (3)/(2) overflow, wirelength, via cuts
    ev_res, ev_ms = None, None
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            A.profiling(True)
            A.profile(reset=True)
        ev_res = A.eval_overflow()
    pe = A.profile(reset=True)
    A.profiling(False)
    ev_ms = pe["eval_ms"] / max(args.steps, 1)
    sol = A.solution()
    via_cuts = int((sol["vias"][:, 3] - sol["vias"][:, 2]).sum()) if len(sol["vias"]) else 0
    st = A.stats()
    value = d.n_nets / (ms / 1000.0)

    # roofline of the dominant kernel (k_assign) from live CUDA-event times over the timed region
    hbm, peak_src = peaks()
    a_bytes, c_bytes, e_bytes = algorithmic_bytes(st, d.L, d.n_nets, via_cuts)
    a_launch = prof["assign_launches"] / args.steps
    a_ms = prof["assign_ms"] / args.steps           # k_assign device time per step (this rank's shard)
    # at world 1 with conflict-free batches the demand commit (K8) runs inside the k_assign launches
    # (fused red.relaxed reductions): its read-modify-write bytes are that kernel's too
    fused = world == 1 and args.batching == "conflict-free"
    a_bytes_rank = (a_bytes + (c_bytes if fused else 0)) / world
    achieved = a_bytes_rank / (a_ms / 1000.0) / 1e9 if a_ms > 0 else None
    ncu = ncu_summary(d.name)
    fp64_peak = la.la_fp64_peak(local_rank)         # FP64 vector pipe, lane ops/s (SURVEY d.3)
    roof = {"kernel": ("k_assign_g (K4+K5 Alg. 3 DP + Alg. 4 backtrack" + (" + fused K8 commit)" if fused else ")")),
            "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": (achieved / hbm) if achieved else None,
            "traffic": ncu.get("dram_bytes_per_launch"), "traffic_source": ncu.get("file"),
            "alg_bytes_per_launch": a_bytes_rank / max(a_launch, 1), "launches_per_step": a_launch,
            "alg_bytes_includes": "K4/K5 per SURVEY d.4" + (" + K8 commit (8 B per unit edge and per via cut)"
                                                             if fused else ""),
            "kernel_ms_per_step": a_ms, "kernel_share_of_step": a_ms / ms,
            "peak_source": peak_src,
            "fp64": {"peak_ops_per_s": fp64_peak, "peak_source": "measured (la_fp64_peak: DADD chains on every SM)",
                     "pipe_active_frac": ncu.get("fp64_pipe_active_frac"),
                     "pipe_active_source": ncu.get("fp64_source"),
                     "issue_active_frac": ncu.get("issue_active_frac")}}
    step_bytes = a_bytes + c_bytes + e_bytes
    roof_step = {"alg_bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms / 1000.0) / 1e9,
                 "frac": step_bytes / (ms / 1000.0) / 1e9 / hbm,
                 "kernel_ms_per_step": {"k_assign": a_ms, "k_commit": prof["commit_ms"] / args.steps,
                                        "k_elmore": prof["elmore_ms"] / args.steps,
                                        "reconcile": prof["reconcile_ms"] / args.steps}}
    # algorithmic bytes: every packed wire / via word once (4 B); the per-layer wirelength and via cuts
    # come from the same histograms unless a value was clamped (R20), when the node pass reads lay, sb,
    # st, edir (u8) and len (i32) per node as well
    ev_bytes = 4 * (int(sum(d.wire_layer_sizes())) + d.X * d.Y * (d.L - 1)) + \
        (8 * st["n_nodes"] if ev_res["out_of_domain"] else 0)
    pre = None if args.no_pre else pre_assignment(args, A, d, la, crit, st, hbm)
    A.close()
    evaluator = {"kernel": "k_eval_plane x3 (NEXT #3: Eq. (3)/(2) overflow; wirelength and via cuts from the "
                           "same histograms)",
                 "bound": "hbm", "ms": ev_ms, "alg_bytes": ev_bytes,
                 "achieved": ev_bytes / (ev_ms / 1000.0) / 1e9 if ev_ms else None, "peak": hbm, "unit": "GB/s",
                 "frac": (ev_bytes / (ev_ms / 1000.0) / 1e9 / hbm) if ev_ms else None,
                 "tof_wire": ev_res["tof_wire"], "legacy_wire": ev_res["legacy_wire"],
                 "via_cuts": ev_res["via_cuts"], "wire_cap_fF": ev_res["wire_cap"],
                 "out_of_domain": ev_res["out_of_domain"]}

    # e2e: the public API from host buffers: init_grid + load_nets + all batches + Elmore + solution to host
    e2e = None
    if not args.no_e2e:
        vals, h2d, d2h = [], 0, 0
        for i in range(args.e2e_steps + 1):
            nid_e = fresh_nccl_id()
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            B = la.LayerAssigner(d, device=local_rank, rank=rank, world=world, nccl_id=nid_e,
                                 stream=stream.cuda_stream)
            B.load(snapshot_batches=snap)
            B.assign_all()
            B.eval_timing()
            B.solution()
            torch.cuda.synchronize()
            barrier()
            dt = time.perf_counter() - t0
            s2 = B.stats()
            B.close()
            if world > 1:
                t = torch.tensor([dt], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t.item())
            if i > 0:          # first pass is a warm-up
                vals.append(dt)
                h2d, d2h = s2["h2d_bytes"], s2["d2h_bytes"]
        e2e = {"value": d.n_nets / statistics.median(vals), "unit": "nets/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "seconds_per_step": statistics.median(vals),
               "includes": "la_init_grid + la_load_nets (host tree build, GPU batching, upload) + every batch + "
                           "la_eval_timing + la_get_solution, pageable host buffers"}

    cpu = cpu2 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(d, args.cpu_seconds)
        cpu2 = cpu_baseline_mode2(d, args.cpu_seconds, cpu["value"])

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "nets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": d.name, "batching": args.batching, "nets": d.n_nets, "grid": f"{d.X}x{d.Y}", "layers": d.L,
                       "pins": d.n_pins, "la_nodes": st["n_nodes"], "wirelength": st["wirelength"],
                       "via_cuts": via_cuts, "batches": nb, "max_height": st["max_height"],
                       "max_batch_nets": st["max_batch_nets"],
                       "parallelism": f"dp{world}: nets of every conflict-free batch sharded over {world} GPU(s)",
                       "l2": f"inputs > L2: {(4 * (st['via_state_words'] + st['wire_state_words']) + 50 * st['n_nodes']) / 1e9:.2f} GB touched per step",
                       "setup_s": setup_s, "load_ms": st0["load_ms"], "batching_ms": st0["batch_ms"]},
            "roofline": roof, "roofline_step": roof_step, "evaluator": evaluator, "pre_assignment": pre,
            "cpu_baseline": cpu, "cpu_baseline_mode2": cpu2, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(out), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

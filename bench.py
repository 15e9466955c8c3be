#!/usr/bin/env python
"""bench.py — DP force-evaluation MD throughput on B200 (contract in the task brief).

Workload (BASELINE.json configs[4], the north-star target box, the largest paper
box): DPA3 analog (make_model(message_passing, 3, 0.6, 2, 8, 32, seed 1)) on the
synthetic 2PTC-shaped protein-in-water box (4114 atoms, generate_synthetic_system
seed 7), velocity-Verlet MD at dt = 1 fs, the exact rc neighbour list of
build_input_periodic every step (filtered out of Verlet candidate rows within
rc + 0.1 nm that the cell-list search rebuilds after an atom moved > 0.05 nm; the
rebuild count of the timed steps is in the line), each step = kick+drift,
neighbour list, full DP energy/force/virial evaluation, kick -- one CUDA graph per
step.  The DPA2 analog
(embed_fit, depth 1) on the same box is measured the same way in the same run and
reported under "models": {"dpa2": {...}} with its own roofline / e2e / cpu_baseline.

  value      steps/s over all ranks (N independent replica boxes = weak scaling),
             each timed step bracketed by CUDA events on the launching stream,
             L2 flushed (256 MiB write) before every step outside the events.
  e2e        the same MD through the host-buffer C-ABI call: a C++ caller runs the
             reference's velocity_verlet_step on host arrays with hmdp_compute as
             its force function (csrc/hmdp_caller_md.cpp), so every step carries
             the H2D of positions/types and the D2H of forces/energy; timed with
             CUDA events around the loop.
  roofline   dominant kernel (ncu launch-list share of the step x the live step
             time); achieved = the FLOPs that kernel executes per launch / its
             duration; peak = FP32 FFMA throughput measured here (the kernels are
             FP32 SIMT, parity-mode precision).  Beside it: the SURVEY §8(d)
             reference-counter rate of the same kernel and the step-level roofline
             of record (t_lb = FLOP_alg / peak vs the measured step).
  cpu_baseline  the reference compiled from its own sources (oracle/_ref), same
             MD workload, one replica per host thread.

  --impl reference   times only the reference CPU path (rank 0) on the same workload.
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

# name -> (family, depth): the reference's two toy families (DPA2 / DPA3 analogs)
# and the DeePMD-style families of the north star (no reference function,
# DESIGN.md §11): se_a (smooth env matrix, G^T R R^T G) and a 2-layer repformer
# (DPA2-style gated neighbour self-attention), 2-layer repflow (DPA3-style
# edge/angle message passing).
MODELS = {"dpa2": (0, 1), "dpa3": (1, 3), "se_a": (2, 1), "repformer": (3, 3), "repflow": (4, 3)}


def make_bench_model(P, name):
    fam, depth = MODELS[name]
    if fam >= 2:
        return P.make_dp_model(P.ModelFamily(fam), depth, 0.6, 0.3, 2, 1)
    return P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, 1)
SYSTEMS = {"1YRF": 582, "1UBQ": 1231, "3LZM": 2643, "2PTC": 4114}
METRIC = "DPA2/DPA3 force-eval steps/s & ns/day at 1/2/4/8 B200 vs CPU ref; %roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", choices=list(MODELS), default="dpa3")
    ap.add_argument("--system", choices=list(SYSTEMS), default="2PTC")
    ap.add_argument("--also", type=str, default="dpa2",
                    help="further models measured on the same system, reported under "
                         "\"models\" in the same JSON line ('' = none)")
    ap.add_argument("--replicas", type=str, default="1,1,1", help="periodic replication per rank")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--strong", action="store_true",
                    help="--mode dd: split ONE box over the ranks (strong scaling, SURVEY "
                         "§8(d) configs 3/4) instead of one box per rank")
    ap.add_argument("--mode", choices=["dd", "dd-gather", "dd-allreduce", "replicas"], default="dd",
                    help="N>1: halo-exchange spatial domain decomposition of the box "
                         "replicated over the rank grid (default; point-to-point NCCL halo "
                         "rounds, one CUDA graph per MD step), the paper's gather-to-root "
                         "strategy on the same engine (dd-gather), the replicated all-reduce "
                         "variant for tiny boxes (dd-allreduce), or independent replica "
                         "boxes (replicas)")
    return ap.parse_args()


def ns_per_day(steps_per_s, dt_fs=1.0):
    return steps_per_s * dt_fs * 1e-6 * 86400.0


# ---------------------------------------------------------------------------
# algorithmic FLOPs per kernel: the reference counter (inference.cpp:389-414)
# split along our kernel boundaries; the sum over kernels equals the counter.
# ---------------------------------------------------------------------------
def mlp_flops(sizes):
    return sum(2 * a * b + 4 * b for a, b in zip(sizes[:-1], sizes[1:]))


def dp_kernel_flops(d, n, ne, m2):
    """Algorithmic FLOPs per kernel of the DeePMD-style families (hmdp_dp.cu), in
    the reference counter's convention (forward, reverse = 2x forward): env
    matrix 30/edge, per-edge embedding MLP, R^T G (8H/edge), G^T R R^T G, MLPs by
    mlp_flops; repformer attention 4H+5 per neighbour pair (m2 = sum_i n_i^2)."""
    H = d["hidden"]
    ax = d["axis"]
    fe = mlp_flops(d["embeddings"][0]["sizes"])
    ff = mlp_flops(d["fitting"]["sizes"])
    desc = ne * (30 + fe + 8 * H) + n * (2 * ax * 4 * H)
    if d["family"] == "se_a":
        return {"sea": 3 * desc + 3 * n * ff}
    fmap = mlp_flops(d["g1map"]["sizes"])
    lay = d["layers"][0]
    fq = mlp_flops(lay["v"]["sizes"])
    fu = mlp_flops(lay["update"]["sizes"])
    if d["family"] == "repflow":  # v, o projections; per angle pair 3 + 4H (tanh counted once)
        fwd = ne * (2 * fq + 6 * H) + m2 * (3 + 4 * H) + n * (fq + 2 * 3 * ax * H + fu)
    else:
        fwd = ne * (4 * fq + 6 * H) + m2 * (4 * H + 5) + n * (fq + 2 * 3 * ax * H + fu)
    emb = desc + n * fmap
    return {"rf_embed": emb, "rf_fwd": fwd, "rf_top": 3 * fwd + 3 * n * ff, "rf_bwd": 2 * fwd,
            "rf_embed_bwd": 2 * emb}


def kernel_flops(model_dict, n, n_owned, ne, m2=0):
    if model_dict["family"] in ("se_a", "repformer", "repflow"):
        return dp_kernel_flops(model_dict, n, ne, m2)
    H = model_dict["hidden"]
    K = len(model_dict["basis"]["centers"])
    fe = mlp_flops(model_dict["embedding"]["sizes"])
    ff = mlp_flops(model_dict["fitting"]["sizes"])
    layers = model_dict["layers"]
    M = len(layers)
    out = {}
    if M == 0:
        out["embed_fit"] = ne * (20 + 10 * K) + 3 * n * fe + 3 * n_owned * ff
        return out
    fm = [mlp_flops(l["message"]["sizes"]) for l in layers]
    fu = [mlp_flops(l["update"]["sizes"]) for l in layers]
    # split along the kernel boundaries of the pull-form periodic path (hmdp_net.cu):
    # msg_fwd_last = top layer forward + fitting + the top update MLP's backward;
    # msg_bwd(l) = layer l+1's per-edge backward (at the senders) + layer l's update
    # backward; embed_bwd = layer 0's per-edge backward + the embedding backward
    ebwd = [ne * (2 * fm[l] + 6 * H + 3 * K) for l in range(M)]
    ubwd = [n * (2 * fu[l] + 2 * H) for l in range(M)]
    out["embed"] = ne * (20 + 10 * K) + n * fe
    out["msg_fwd"] = sum(ne * fm[l] + n * fu[l] for l in range(M - 1)) / max(M - 1, 1)
    out["msg_fwd_last"] = ne * fm[-1] + n * fu[-1] + 3 * n_owned * ff + ubwd[-1]
    out["msg_bwd"] = sum(ebwd[l + 1] + ubwd[l] for l in range(M - 1)) / max(M - 1, 1)
    out["embed_bwd"] = ebwd[0] + 2 * n * fe
    return out


# launches per MD step of each kernel name (msg_fwd / msg_bwd: M - 1 each)
M_LAUNCH = {"msg_fwd": lambda d: max(len(d.get("layers", [])) - 1, 0),
            "msg_bwd": lambda d: max(len(d.get("layers", [])) - 1, 0)}


def exec_kernel_flops(model_dict, n, n_owned, ne, pull=1):
    """FLOPs our kernels execute per launch (FMA = 2), i.e. the algorithm as restructured
    (per-atom P rows, msum through W2 once per atom, the per-edge message
    backward as rank-1 terms) rather than the reference's per-edge MLPs.  Per edge and
    layer: forward 2KH (W1b b) + 5H (tanh, add) + 2H (s z accumulate); backward 2KH
    (W1b^T b') + 10H (dz, sums, dE/dr terms) [+ 2KH + 5H recomputing z, pull = 2].  Per
    atom: every mat-vec 2 in out (+ activation 4 out, as the reference's counter)."""
    if model_dict["family"] in ("se_a", "repformer", "repflow"):
        return None
    H = model_dict["hidden"]
    K = len(model_dict["basis"]["centers"])
    mv = lambda i, o, act=False: 2 * i * o + (4 * o if act else o)  # noqa: E731
    M = len(model_dict["layers"])
    e_rad = ne * (20 + 10 * K)
    e_fwd = ne * (2 * K * H + 7 * H + 1)
    e_bwd = ne * (2 * K * H + 10 * H + 2 + (2 * K * H + 5 * H if pull == 2 else 0))
    emb_f = mv(32, H, True) + mv(H, H)
    emb_b = mv(H, H) + mv(H, 32) + H
    fit = mv(H, H, True) + 2 * H + mv(H, H) + H  # forward, head, backward
    upd_f = mv(H, H) + mv(2 * H, H, True) + mv(H, H) + H  # msum W2, update MLP, residual
    upd_b = mv(H, H) + mv(H, 2 * H) + mv(H, H) + 2 * H  # W2u^T, W1u^T, W2^T (v), c0
    out = {}
    if M == 0:
        out["embed_fit"] = e_rad + ne * 2 * K + n * (emb_f + emb_b) + n_owned * fit
        return out
    out["embed"] = e_rad + ne * K + n * (emb_f + mv(H, H))
    out["msg_fwd"] = e_fwd + n * (upd_f + mv(H, H))
    out["msg_fwd_last"] = e_fwd + n * (upd_f + upd_b) + n_owned * fit
    out["msg_bwd"] = e_bwd + n * (mv(H, H) + upd_b)
    out["embed_bwd"] = e_bwd + ne * 2 * K + n * (mv(H, H) + emb_b)
    return out


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.rows = []
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                s, m, u = float(r[0]), float(r[1]), float(r[2])
            except ValueError:
                continue
            mx.append(m)
            if u > 0:
                sm.append(s)
            for k, name in enumerate(names):
                if r[3 + k].lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# Workload identity shared by both arms (the driver compares the config dicts)
# ---------------------------------------------------------------------------
def workload_config(args, model_name, world):
    n = SYSTEMS[args.system]
    reps = tuple(int(v) for v in args.replicas.split(","))
    n_rep = reps[0] * reps[1] * reps[2]
    return {"workload": f"{model_name.upper()} velocity-Verlet MD step on the {args.system}-shaped "
                        f"box (dt 1 fs, exact rc neighbour list every step, E+F+W every step)",
            "model": model_name, "system": args.system, "atoms": n * n_rep,
            "replicas_per_rank": list(reps), "precision": args.precision,
            "parallelism": f"replicas x{world}"}


def replicate_np(x, t, m, v, box, reps):
    """Periodic replica box, numpy only (the reference arm must not load libhmdp)."""
    import numpy as np

    rx, ry, rz = reps
    sh = np.array([(i, j, k) for k in range(rz) for j in range(ry) for i in range(rx)], float) * box
    r = sh.shape[0]
    return ((x[None] + sh[:, None]).reshape(-1, 3), np.tile(t, r), np.tile(m, r),
            np.tile(v, (r, 1)), box * np.array(reps, float))


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref): P concurrent replicas of the same MD workload
# ---------------------------------------------------------------------------
def reference_md(model_name, system, steps, warmup, precision, threads, replicas=(1, 1, 1)):
    import numpy as np

    import oracle as O

    fam, depth = MODELS[model_name]
    if fam >= 2:
        # no reference implementation exists for the DeePMD-style families: the
        # FP64 oracle (torch autograd on the host cores) is the CPU path
        import torch

        import paper_2602_02234_b200 as P
        from oracle import dpfamily as DF

        s = P.generate_synthetic_system(SYSTEMS[system])
        if tuple(replicas) != (1, 1, 1):
            s = P.replicate(s, replicas)
        torch.set_num_threads(threads)
        m = make_bench_model(P, model_name).as_dict()
        x, v = s.positions.copy(), s.velocities.copy()
        half, dt = 0.0005, 0.001

        def force(x):
            return DF.evaluate(m, s.types, *O.neighbors(x, s.box, 0.6))["forces"]

        f = force(x)
        t0 = time.perf_counter()
        for _ in range(steps):
            v += f * (half / s.masses[:, None])
            x += v * dt
            f = force(x)
            v += f * (half / s.masses[:, None])
        wall = time.perf_counter() - t0
        return steps / wall, wall, "port"
    # the reference's own generator and model (oracle/_ref): libhmdp is never loaded here
    x, t, m, v, box = O.ref_synthetic(SYSTEMS[system])
    if tuple(replicas) != (1, 1, 1):
        x, t, m, v, box = replicate_np(x, t, m, v, box, replicas)
    if O.ref_available():
        rm = O.RefModel(O.ref_model_json(fam, depth))
        if warmup:
            O.ref_md(rm, x, v, t, m, box, prec=precision, steps=warmup, threads=threads)
        wall, _, _, _ = O.ref_md(rm, x, v, t, m, box, prec=precision, steps=steps, threads=threads)
        return steps * threads / wall, wall, "reference"
    raise SystemExit("reference arm needs oracle/_ref (built from /root/reference by build())")


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_line(args, model_name, world, budget_s):
    threads = cpu_count()
    # bounded sample: calibrate the per-step cost on a few steps, then time as many of
    # the K requested steps as fit in ~budget_s of wall (the whole run stays within
    # minutes for any K; the rate, not the step count, is the measurement)
    reps = tuple(int(v) for v in args.replicas.split(","))
    cal = min(args.steps, 2)
    _, wall0, _ = reference_md(model_name, args.system, cal, 0, args.precision, threads, reps)
    timed = max(cal, min(args.steps, int(budget_s / max(wall0 / cal, 1e-6))))
    sps, wall, kind = reference_md(model_name, args.system, timed, min(args.warmup, 1),
                                   args.precision, threads, reps)
    cfg = workload_config(args, model_name, world)
    sample = (f"{model_name} {args.system} ({cfg['atoms']} atoms) velocity-Verlet MD, {timed} timed "
              f"steps per replica (of the {args.steps} requested; ~{budget_s:.0f} s cap) x {threads} "
              f"concurrent replicas (one per host thread), {args.precision}")
    return {
        "metric": METRIC, "value": sps, "unit": "steps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / sps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (generate_synthetic_system seed 7), random-init weights (seed 1)",
        "config": cfg,
        "impl": "reference",
        "ns_per_day": ns_per_day(sps),
        "cpu_baseline": {"value": sps, "unit": "steps/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": sps, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference(args, rank, world):
    if rank != 0:
        return
    line = reference_line(args, args.model, world, 45.0)
    extra = [m for m in args.also.split(",") if m and m != args.model]
    if extra:
        line["models"] = {m: reference_line(args, m, world, 30.0) for m in extra}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
SHARES = os.path.join(ROOT, "profiles", "round2", "launch_shares.json")


def ncu_shares(model_name, system):
    """Per-kernel share of one MD step from the committed ncu launch list of this bench
    workload (tools/launch_shares.py; serialised, so only the SHARES are used)."""
    try:
        return json.load(open(SHARES))[model_name][system]
    except Exception:
        return None


def measure(args, model_name, rank, world, local_rank, dist, stream, flush, with_cpu):
    """One model on the bench system: the timed device MD loop (headline value), the
    per-kernel roofline, the warm-L2 context figure, the host-buffer e2e leg and the
    CPU baseline.  Returns the JSON fields of that model's line (rank 0)."""
    import ctypes

    import numpy as np
    import torch

    import paper_2602_02234_b200 as P
    from paper_2602_02234_b200._lib import check, lib, ptr
    from paper_2602_02234_b200.md import DeviceMD

    dev = torch.device("cuda", local_rank)
    L = lib()
    prec = P.Precision[args.precision]
    model = make_bench_model(P, model_name)
    s = P.generate_synthetic_system(SYSTEMS[args.system])
    reps = tuple(int(v) for v in args.replicas.split(","))
    if reps != (1, 1, 1):
        s = P.replicate(s, reps)
    n = s.n_atoms
    ctx = P.Context(model, device=local_rank, max_atoms=n)
    check(L.hmdp_set_stream(ctx.handle, ctypes.c_void_p(stream.cuda_stream)))
    inp = P.build_input_periodic(s.positions, s.types, np.arange(n), s.box, 0.6, device=local_rank)
    ne = int(inp.edge_offset[-1])
    m2 = int(np.sum(np.diff(inp.edge_offset).astype(np.int64) ** 2))
    # per MD step: search + network + force (the cell binning and both velocity-Verlet
    # halves are fused into the force kernel; kernels_per_eval counts the binning)
    per_step_kernels = ctx.kernels_per_eval() - 1

    sampler = ClockSampler(local_rank) if rank == 0 else None
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, 0.001, prec,
                  steps_per_graph=1)
    enqueue = L.hmdp_md_enqueue
    for _ in range(max(args.warmup, 3)):
        check(enqueue(md.handle, 1))
    torch.cuda.synchronize(dev)
    check(L.hmdp_check(ctx.handle))
    skin_nm, rebuilds0 = md.stats()

    # ---- timed region: one graph launch per MD step, L2 flushed between steps ----
    K = args.steps
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    wall0 = time.perf_counter()
    for k in range(K):
        flush.zero_()
        ev0[k].record(stream)
        check(enqueue(md.handle, 1))
        ev1[k].record(stream)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - wall0
    if dist:
        dist.barrier()
    t_ms = float(sum(a.elapsed_time(b) for a, b in zip(ev0, ev1)))
    check(L.hmdp_md_get(md.handle, None, None, None, None))  # latched device errors
    rebuilds = md.stats()[1] - rebuilds0
    if dist:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = world * K / (t_ms * 1e-3)
    ms_step = t_ms / K

    # ---- warm-L2 multi-step graph (context, not the headline): 100 steps per graph
    # launch, no flush; warmed up before timing so graph capture and clock ramp are
    # outside the events ----
    md_warm = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, 0.001, prec,
                       steps_per_graph=100)
    check(enqueue(md_warm.handle, 300))
    torch.cuda.synchronize(dev)
    KW = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    check(enqueue(md_warm.handle, KW))
    e1.record(stream)
    torch.cuda.synchronize(dev)
    warm_sps = KW / (e0.elapsed_time(e1) * 1e-3)
    md_warm.close()

    # ---- per-kernel event timing (an event node after every kernel inside the step
    # graph: breaks the PDL overlap, so these are upper bounds on kernel time) ----
    check(L.hmdp_profile(ctx.handle, 1))
    md_prof = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, 0.001, prec,
                       steps_per_graph=1)
    KP = min(K, 100)
    sums: dict[str, float] = {}
    counts: dict[str, int] = {}
    buf = (ctypes.c_float * 64)()
    cnt = ctypes.c_int()
    for k in range(KP + 5):
        flush.zero_()
        check(enqueue(md_prof.handle, 1))
        check(L.hmdp_profile_read(ctx.handle, buf, 64, ctypes.byref(cnt)))
        if k < 5:
            continue
        for i in range(cnt.value):
            name = L.hmdp_profile_name(ctx.handle, i).decode()
            sums[name] = sums.get(name, 0.0) + buf[i]
            counts[name] = counts.get(name, 0) + 1
    check(L.hmdp_profile(ctx.handle, 0))
    md_prof.close()
    if sampler:
        clocks = sampler.stop()
    event_ms = {k: sums[k] / counts[k] for k in sums}
    kflops = kernel_flops(model.as_dict(), n, n, ne, m2)  # SURVEY §8(d) reference counter
    # our algorithm's FLOPs per launch (the z rows are recomputed beyond ~48 MB of rows,
    # hmdp_net.cu pull_mode: ~6 k atoms for the 2-layer model)
    pull = 2 if n * max(len(model.as_dict().get("layers", [])), 1) * 32 * 32 * 4 > 48 * 2**20 else 1
    xflops = exec_kernel_flops(model.as_dict(), n, n, ne, pull)
    # per-kernel duration inside the timed loop = its ncu share of the step x the live
    # ms_per_step (PDL overlap intact); the event-timed durations are the fallback
    shares = ncu_shares(model_name, args.system) if reps == (1, 1, 1) else None
    if shares and all(k in shares for k in kflops if k in event_ms):
        kern_ms = {k: shares[k] * ms_step for k in shares}
        dur_src = (f"ncu launch-list share of the step ({os.path.relpath(SHARES, ROOT)}) x the "
                   f"live ms_per_step")
    else:
        kern_ms = event_ms
        dur_src = "CUDA events around every kernel in the step graph (PDL broken: upper bound)"
    cands = {k: v for k, v in kern_ms.items() if k in kflops}
    tmax = max(cands.values())
    dom = max((k for k in cands if cands[k] >= 0.97 * tmax), key=lambda k: kflops[k])
    peak = ctypes.c_double()
    check(L.hmdp_peak_fp32(local_rank, 200, ctypes.byref(peak)))
    peak_tc = ctypes.c_double()  # 3xTF32 mma.sync: the DeePMD-family projections' pipe
    check(L.hmdp_peak_tf32x3(local_rank, 200, ctypes.byref(peak_tc)))
    peak_umma = ctypes.c_double()  # tcgen05 kind::tf32 raw (3xTF32 delivers a third)
    check(L.hmdp_peak_tcgen05_tf32(local_rank, 100, ctypes.byref(peak_umma)))
    # roofline of the dominant kernel on the FLOPs our kernels execute (<= peak); the
    # reference-counter rate beside it exceeds the peak where the restructured
    # algorithm needs fewer FLOPs than the reference's per-edge MLPs
    fl = xflops if xflops else kflops
    achieved = fl[dom] / (kern_ms[dom] * 1e-3) / 1e12
    ref_rate = kflops[dom] / (kern_ms[dom] * 1e-3) / 1e12
    # step-level roofline of record: t_lb = FLOP_alg(step) / peak
    flop_alg_step = sum(kflops[k] * (M_LAUNCH.get(k, 1)(model.as_dict()) if callable(M_LAUNCH.get(k)) else 1)
                        for k in kflops)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "round2", "ncu_traffic.json")
    if not os.path.exists(tfile):
        tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(model_name, {}).get(args.system, {}).get(dom)
        except Exception:
            traffic = None
    mp = {}
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        try:
            mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            mp = {}

    # ---- e2e: host-buffer C-ABI provider driven by a C++ caller running the
    # reference's velocity_verlet_step (csrc/hmdp_caller_md.cpp) ----
    KE = min(K, 300)
    prov_ctx = P.Context(model, device=local_rank, max_atoms=n)
    check(L.hmdp_set_stream(prov_ctx.handle, ctypes.c_void_p(stream.cuda_stream)))
    caller = ctypes.CDLL(os.path.join(ROOT, "paper_2602_02234_b200", "lib", "libhmdp_caller.so"))
    vv = caller.hmdp_caller_velocity_verlet
    vv.restype = ctypes.c_int
    xh = np.ascontiguousarray(s.positions, dtype=np.float64).copy()
    th = np.ascontiguousarray(s.types, dtype=np.int32)
    vh = np.ascontiguousarray(s.velocities, dtype=np.float64).copy()
    mh = np.ascontiguousarray(s.masses, dtype=np.float64)
    bh = np.ascontiguousarray(s.box, dtype=np.float64)
    out = prov_ctx.compute(xh, th, bh, prec)
    fh = np.ascontiguousarray(out.forces).copy()
    eh = ctypes.c_double()
    vv_args = (prov_ctx.handle, ctypes.c_int(n), ptr(xh), ptr(vh), ptr(fh), ptr(th), ptr(bh),
               ptr(mh), ctypes.c_double(0.001), None, ctypes.c_int(int(prec)), ctypes.byref(eh))
    check(vv(*vv_args[:9], ctypes.c_int(5), *vv_args[10:]))  # warm-up (graph captured)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    check(vv(*vv_args[:9], ctypes.c_int(KE), *vv_args[10:]))
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1)
    if dist:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = world * KE / (e2e_ms * 1e-3)
    h2d = xh.nbytes + th.nbytes
    d2h = fh.nbytes + 11 * 8
    prov_ctx.close()
    md.close()
    ctx.close()

    if rank != 0:
        return None
    cpu = None
    if with_cpu:
        threads = cpu_count()
        # bounded sample: ~cpu_seconds of wall on all host threads
        per_step = {"dpa3": 0.2, "dpa2": 0.012, "se_a": 0.03, "repformer": 0.06,
                    "repflow": 0.06}[model_name]
        per_step *= n / 582
        steps_cpu = max(2, int(args.cpu_seconds / per_step))
        sps, cwall, kind = reference_md(model_name, args.system, steps_cpu, 1, args.precision,
                                        threads, reps)
        if MODELS[model_name][0] >= 2:
            sample = (f"{steps_cpu} MD steps of one {n}-atom box through the FP64 torch oracle "
                      f"(no reference implementation of this family), {threads} threads, "
                      f"{cwall:.1f} s wall")
        else:
            sample = (f"{steps_cpu} MD steps x {threads} concurrent replicas of the same "
                      f"{n}-atom box (the reference compiled from its sources), "
                      f"{args.precision}, {cwall:.1f} s wall")
        cpu = {"value": sps, "unit": "steps/s", "cores": threads, "kind": kind, "sample": sample}

    return {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (generate_synthetic_system seed 7), random-init weights (seed 1)",
        "config": workload_config(args, model_name, world),
        "verlet": {"skin_nm": skin_nm, "rebuilds_in_timed_steps": rebuilds, "timed_steps": K,
                   "note": "every step filters the exact rc list (bitwise the full search's, "
                           "tests/test_gpu_skin.py) out of candidate rows within rc + skin; "
                           "the rows are rebuilt by the cell-list search on the steps counted"},
        "workload_detail": {"edges": ne, "graph": "one CUDA graph launch per MD step",
                            "l2": "flushed (256 MiB write) before every timed step, outside "
                                  "the events"},
        "ns_per_day": ns_per_day(value),
        "warm_l2_graph100": {"steps_per_s": warm_sps, "ns_per_day": ns_per_day(warm_sps),
                             "note": f"{KW} steps in 100-step graphs after a 300-step warm-up, "
                                     f"L2 not flushed, 1 rank"},
        "roofline": {"bound": "fp32-simt", "achieved": achieved, "peak": peak.value,
                     "unit": "TFLOP/s", "frac": achieved / peak.value, "traffic": traffic,
                     "kernel": dom, "flops_per_launch": fl[dom],
                     "flops_basis": "FLOPs the restructured kernels execute (bench.exec_kernel_flops, "
                                    "DESIGN.md §7)" if xflops else "reference counter",
                     "ref_counter": {"flops_per_launch": kflops[dom], "tflops": ref_rate,
                                     "frac": ref_rate / peak.value,
                                     "note": "SURVEY §8(d) FLOP_alg (the reference's per-edge MLP "
                                             "counter, inference.cpp:389-402) over the same "
                                             "duration; > 1 means the kernel beats the "
                                             "reference algorithm's FP32 roofline"},
                     "step": {"flop_alg_per_step": flop_alg_step,
                              "t_lb_us": flop_alg_step / (peak.value * 1e12) * 1e6,
                              "t_step_us": ms_step * 1e3,
                              "frac": flop_alg_step / (peak.value * 1e12) / (ms_step * 1e-3),
                              "note": "SURVEY §8(d) roofline of record for the whole MD step: "
                                      "t_lb = FLOP_alg / P_fp32 vs the measured step"},
                     "mean_launch_us": kern_ms[dom] * 1e3, "duration_source": dur_src,
                     "peak_kind": "measured FP32 FFMA (SIMT) throughput on this GPU "
                                  "(hmdp_peak_fp32): the parity-mode kernels run FP32 FMA",
                     "frac_of_bf16_tensor_peak": achieved / mp["bf16_tflops"] if "bf16_tflops" in mp else None,
                     "peak_tf32x3_tflops": peak_tc.value,
                     "peak_tcgen05_tf32_raw_tflops": peak_umma.value,
                     "peak_tcgen05_tf32x3_tflops": peak_umma.value / 3.0,
                     "tcgen05_note": "the dense atom-level MLPs on tcgen05 (3xTF32, TMEM) lose the "
                                     "A/B at every measured size (profiles/round2/tcgen05.md); "
                                     "the fused FP32 SIMT kernels are the default",
                     "frac_per_kernel": {k: fl[k] / (cands[k] * 1e-3) / 1e12 / peak.value
                                         for k in sorted(cands, key=lambda k: -cands[k])}},
        "kernels_us": {k: v * 1e3 for k, v in sorted(kern_ms.items(), key=lambda kv: -kv[1])},
        "kernels_event_us": {k: v * 1e3 for k, v in sorted(event_ms.items(), key=lambda kv: -kv[1])},
        "gpu_launches": per_step_kernels * K,
        "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "C++ caller: velocity_verlet_step (integrators.cpp:32-47) on host arrays, "
                        "force function = hmdp_compute (host xyz/types in, forces/E out)"},
        "cpu_baseline": cpu,
        "clocks": clocks if sampler else None,
        "wall_s_timed_region": wall,
    }


def run_ours(args, rank, world, local_rank, dist):
    import torch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # one explicit (non-default) stream carries everything: torch's L2 flush and
    # CUDA events, and every libhmdp launch (hmdp_set_stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    with_cpu = world == 1 and not args.no_cpu_baseline
    line = measure(args, args.model, rank, world, local_rank, dist, stream, flush, with_cpu)
    extra = [m for m in args.also.split(",") if m and m != args.model]
    models = {}
    for m in extra:
        models[m] = measure(args, m, rank, world, local_rank, dist, stream, flush, with_cpu)
    if rank != 0:
        return
    if models:
        line["models"] = models
    print(json.dumps(line), flush=True)


def run_gdd(args, rank, world, local_rank, dist):
    """N > 1, --mode dd (default DD path): device-resident domain decomposition
    (hmdp_gdd_*).  Global box = the per-rank box replicated over the rank grid (one
    box per GPU, weak scaling); every step = roles + neighbour list of this rank's
    owned + halo atoms, the network over its owned atoms, and the per-layer halo
    exchanges as fixed-size SUM all-reduces (NCCL) — the whole MD step (velocity
    Verlet on the replicated positions included) captured in ONE CUDA graph per
    rank, collectives inside.  value = world * steps / max-over-ranks time."""
    import numpy as np
    import torch

    import paper_2602_02234_b200 as P
    from paper_2602_02234_b200 import dd

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    prec = P.Precision[args.precision]
    model = make_bench_model(P, args.model)
    if model.is_dp():
        raise SystemExit("--mode dd: the DeePMD-style families run replicas only (DESIGN.md §11)")
    base = P.generate_synthetic_system(SYSTEMS[args.system])
    dims = dd.rank_grid(world)
    s = base if args.strong else P.replicate(base, dims)
    boxes = 1 if args.strong else world
    n = s.n_atoms
    eng = dd.DeviceDD(P.Context(model, device=local_rank, max_atoms=n), n, s.types, s.box, dims,
                      rank, prec, masses=s.masses)
    eng.load(s.positions, s.velocities)
    use_graph = dist.get_backend() == "nccl" and not os.environ.get("BENCH_DD_NOGRAPH")
    dd.run_dist(eng, "eval")
    torch.cuda.synchronize(dev)
    E = float(eng.out[0])  # energy of the initial configuration (extensivity check)
    dd.run_dist(eng, "open", 0.001)
    for _ in range(max(args.warmup, 3)):
        l0 = eng.launches()
        dd.run_dist(eng, "md", 0.001)
        per_step_kernels = eng.launches() - l0
    torch.cuda.synchronize(dev)
    g = None
    if use_graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                dd.run_dist(eng, "md", 0.001)
            g.replay()
        except Exception as exc:  # symmetric on every rank: all fall back to direct launches
            print(f"rank {rank}: graph capture failed ({exc}); direct launches", file=sys.stderr)
            g = None
            torch.cuda.synchronize(dev)
    # halo share: the same step's collectives timed alone (events, non-graph)
    torch.cuda.synchronize(dev)
    K = args.steps
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        if g is not None:
            g.replay()
        else:
            dd.run_dist(eng, "md", 0.001)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    t_ms = e0.elapsed_time(e1)
    ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # same sizes as the step's collectives, on scratch copies (the engine's state stays intact)
    M = model.depth() - 1  # P^l forward rounds, halo-sum backward rounds, then forces + (E, W)
    bufs = [b.clone() for b in [eng.p] * M + [eng.sg] * M + [eng.fo]]
    ca.record(stream)
    for _ in range(20):
        for b in bufs:
            dist.all_reduce(b)
    cb.record(stream)
    torch.cuda.synchronize(dev)
    halo_ms = ca.elapsed_time(cb) / 20
    # e2e: every step the positions come in from pinned host memory and the step's
    # result (positions, forces, E/W) goes back to pinned host memory, read by the host
    KE = min(K, 300)
    x_h = torch.empty_like(eng.pos, device="cpu").pin_memory()
    fo_h = torch.empty_like(eng.fo, device="cpu").pin_memory()
    x_h.copy_(eng.pos)
    dist.barrier()
    torch.cuda.synchronize(dev)
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    e_host = 0.0
    for _ in range(KE):
        eng.pos.copy_(x_h, non_blocking=True)
        if g is not None:
            g.replay()
        else:
            dd.run_dist(eng, "md", 0.001)
        x_h.copy_(eng.pos, non_blocking=True)
        fo_h.copy_(eng.fo, non_blocking=True)
        stream.synchronize()
        e_host += float(fo_h[3 * n])  # the host reads the step's energy
    eb.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = ea.elapsed_time(eb)
    tt = torch.tensor([t_ms, halo_ms, e2e_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms, halo_ms, e2e_ms = float(tt[0]), float(tt[1]), float(tt[2])
    value = boxes * K / (t_ms * 1e-3)
    e2e_value = boxes * KE / (e2e_ms * 1e-3)
    counts = eng.counts()
    from paper_2602_02234_b200._lib import check, lib

    check(lib().hmdp_check(eng.ctx.handle))
    if rank != 0:
        return
    e_single = P.Context(model, device=local_rank).compute(base.positions, base.types, base.box,
                                                           P.Precision.fp64).energy
    line = {
        "metric": METRIC, "value": value, "unit": f"steps/s ({args.system}-box equivalents)",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": t_ms / K,
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (generate_synthetic_system seed 7), random-init weights (seed 1)",
        "config": {"workload": f"{args.model.upper()} domain-decomposed MD step, " + (
                       f"one {args.system} box split over {dims}" if args.strong else
                       f"{args.system} box replicated {dims} (one box per GPU)"),
                   "model": args.model, "system": args.system, "atoms_total": n,
                   "rank_grid": list(dims), "precision": args.precision,
                   "parallelism": f"device-resident spatial DD x{world}: owner/halo lists on the "
                                  f"device, per-layer rc-halo exchange as SUM all-reduces (NCCL), "
                                  f"replicated velocity Verlet",
                   "graph": "one CUDA graph per MD step incl. NCCL" if g is not None else "none",
                   "rank0_owned": counts[0], "rank0_halo": counts[1]},
        "ns_per_day_per_box": ns_per_day(value / boxes),
        "halo": {"ms_per_step": halo_ms, "rounds_per_step": len(bufs),
                 "share": halo_ms / (t_ms / K)},
        "extensivity": {"E_total": E, "E_single_box_x_boxes": e_single * boxes,
                        "rel_diff": abs(E - e_single * boxes) / abs(e_single * boxes)},
        "gpu_launches": per_step_kernels * K,
        "e2e": {"value": e2e_value, "unit": "steps/s",
                "h2d_bytes_per_step": int(x_h.numel() * 8),
                "d2h_bytes_per_step": int((x_h.numel() + fo_h.numel()) * 8),
                "path": "per step and rank: positions H2D from pinned host memory, the "
                        "captured DD step, positions + forces + (E, W) D2H, host sync"},
    }
    print(json.dumps(line), flush=True)


def run_halo(args, rank, world, local_rank, dist):
    """N > 1, --mode dd (default): the halo-exchange domain decomposition (dd.HaloDD,
    hmdp_gdd_* halo mode).  Global box = the per-rank box replicated over the rank grid
    (weak scaling, one box per GPU) or, with --strong, one box split over the ranks.
    Every rank integrates only the atoms its region owns; each MD step moves exactly
    the halo with point-to-point NCCL rounds to every peer (POS with migration, P^l,
    dE/dh partial sums, partial forces, (E, W) partials) issued from C++ on the
    step's stream, and the whole step -- NCCL included -- is one CUDA graph per rank.
    value = boxes * steps / max-over-ranks time."""
    import numpy as np
    import torch

    import paper_2602_02234_b200 as P
    from paper_2602_02234_b200 import dd

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    prec = P.Precision[args.precision]
    model = make_bench_model(P, args.model)
    if model.is_dp():
        raise SystemExit("--mode dd: the DeePMD-style families run replicas only (DESIGN.md §11)")
    base = P.generate_synthetic_system(SYSTEMS[args.system])
    dims = dd.rank_grid(world)
    s = base if args.strong else P.replicate(base, dims)
    boxes = 1 if args.strong else world
    n = s.n_atoms
    strategy = "gather" if args.mode == "dd-gather" else "halo"
    eng = dd.HaloDD(P.Context(model, device=local_rank, max_atoms=n), n, s.types, s.box, dims,
                    rank, prec, masses=s.masses, stream=stream, strategy=strategy)
    use_nccl = dist.get_backend() == "nccl"
    if use_nccl:  # our own communicator: the C++ engine issues ncclSend/ncclRecv itself
        import ctypes

        from paper_2602_02234_b200._lib import check, lib

        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            check(lib().hmdp_nccl_unique_id(uid))
        obj = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.attach_nccl(obj[0])
    else:  # dry run with ranks sharing a GPU (BENCH_DD_BACKEND=gloo)
        dd.gloo_exchange(eng)
    eng.load(s.positions, s.velocities)
    eng.step("eval")
    E = eng.energy_virial()[0]  # energy of the initial configuration (extensivity check)
    eng.step("open", 0.001)
    for _ in range(max(args.warmup, 3)):
        l0 = eng.launches()
        eng.step("md", 0.001)
        per_step_kernels = eng.launches() - l0
    torch.cuda.synchronize(dev)
    g = None
    if use_nccl and not os.environ.get("BENCH_DD_NOGRAPH"):
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                eng.step("md", 0.001)
            g.replay()
        except Exception as exc:  # symmetric on every rank: all fall back to direct launches
            print(f"rank {rank}: graph capture failed ({exc}); direct launches", file=sys.stderr)
            g = None
    torch.cuda.synchronize(dev)
    K = args.steps
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        if g is not None:
            g.replay()
        else:
            eng.step("md", 0.001)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    t_ms = e0.elapsed_time(e1)
    stats = eng.halo_stats()
    # e2e: every step the positions come in from pinned host memory and the step's
    # result (positions, forces, (E, W)) goes back to pinned host memory, read by the host
    KE = min(K, 300)
    x_h = torch.empty_like(eng.pos, device="cpu").pin_memory()
    f_h = torch.empty_like(eng.f, device="cpu").pin_memory()
    o_h = torch.empty_like(eng.out, device="cpu").pin_memory()
    x_h.copy_(eng.pos)
    dist.barrier()
    torch.cuda.synchronize(dev)
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    e_host = 0.0
    for _ in range(KE):
        eng.pos.copy_(x_h, non_blocking=True)
        if g is not None:
            g.replay()
        else:
            eng.step("md", 0.001)
        x_h.copy_(eng.pos, non_blocking=True)
        f_h.copy_(eng.f, non_blocking=True)
        o_h.copy_(eng.out, non_blocking=True)
        stream.synchronize()
        e_host += float(o_h[0])  # the host reads the step's energy
    eb.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = ea.elapsed_time(eb)
    tt = torch.tensor([t_ms, e2e_ms], dtype=torch.float64, device=dev)
    if use_nccl:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    else:
        tc = tt.cpu()
        dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        tt = tc
    t_ms, e2e_ms = float(tt[0]), float(tt[1])
    value = boxes * K / (t_ms * 1e-3)
    e2e_value = boxes * KE / (e2e_ms * 1e-3)
    roles = eng.roles()
    if rank != 0:
        return
    e_single = P.Context(model, device=local_rank).compute(base.positions, base.types, base.box,
                                                           P.Precision.fp64).energy
    line = {
        "metric": METRIC, "value": value, "unit": f"steps/s ({args.system}-box equivalents)",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": t_ms / K,
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (generate_synthetic_system seed 7), random-init weights (seed 1)",
        "config": {"workload": f"{args.model.upper()} domain-decomposed MD step, " + (
                       f"one {args.system} box split over {dims}" if args.strong else
                       f"{args.system} box replicated {dims} (one box per GPU)"),
                   "model": args.model, "system": args.system, "atoms_total": n,
                   "rank_grid": list(dims), "precision": args.precision,
                   "parallelism": (f"spatial DD x{world}, rc-deep halo exchanged per layer with "
                                   f"point-to-point {'NCCL' if use_nccl else 'gloo'} rounds; owners "
                                   f"integrate their own atoms (migration every step)"
                                   if strategy == "halo" else
                                   f"spatial DD x{world}, gather-to-root (the paper's strategy, "
                                   f"SPEC.md:505): owned atoms -> rank 0 over point-to-point "
                                   f"{'NCCL' if use_nccl else 'gloo'}, one single-domain "
                                   f"evaluation there, forces back to the owners, who integrate"),
                   "graph": "one CUDA graph per MD step incl. NCCL" if g is not None else "none",
                   "rank0_owned": int((roles == 1).sum()), "rank0_halo": int((roles == 2).sum())},
        "ns_per_day_per_box": ns_per_day(value / boxes),
        "halo": {"rounds_per_step": stats["rounds_per_step"],
                 "rank0_halo_bytes_per_step": stats["halo_bytes_per_step"],
                 "rank0_transferred_bytes_per_step": stats["transferred_bytes_per_step"],
                 "packet_capacity_rows": stats["capacity_rows"], "peers": stats["peers"]},
        "extensivity": {"E_total": E, "E_single_box_x_boxes": e_single * boxes,
                        "rel_diff": abs(E - e_single * boxes) / abs(e_single * boxes)},
        "gpu_launches": per_step_kernels * K,
        "e2e": {"value": e2e_value, "unit": "steps/s",
                "h2d_bytes_per_step": int(x_h.numel() * 8),
                "d2h_bytes_per_step": int((x_h.numel() + f_h.numel() + o_h.numel()) * 8),
                "path": "per step and rank: positions H2D from pinned host memory, the "
                        "captured DD step, positions + forces + (E, W) D2H, host sync"},
    }
    print(json.dumps(line), flush=True)


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N
    processes on this node (the driver's own launch sets WORLD_SIZE and skips this)."""
    import socket
    import subprocess

    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    dist = None
    if world > 1:
        import torch.distributed as td

        # BENCH_DD_BACKEND=gloo allows a dry run of the N>1 path with several ranks
        # sharing one GPU (NCCL needs one GPU per rank)
        td.init_process_group(os.environ.get("BENCH_DD_BACKEND", "nccl"), init_method="env://")
        dist = td
        if os.environ.get("BENCH_DD_BACKEND", "nccl") != "nccl":
            import torch

            local_rank = local_rank % max(1, torch.cuda.device_count())
    try:
        # the DeePMD-style families have no domain decomposition: their
        # N > 1 line is N independent replicas
        dd_ok = args.model in ("dpa2", "dpa3")
        if world > 1 and args.mode in ("dd", "dd-gather") and dd_ok:
            run_halo(args, rank, world, local_rank, dist)
        elif world > 1 and args.mode == "dd-allreduce" and dd_ok:
            run_gdd(args, rank, world, local_rank, dist)
        else:
            run_ours(args, rank, world, local_rank, dist)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the B200 Stokes BIO apply (arXiv 1707.06551 hot path).

One step = one pass of every row of SURVEY.md §8(a) over the workload:
bie_apply_SLDL (pack + spectral self term + far-field SL+DL pair sum at every
node) followed by bie_eval_offsurface (velocity + pressure at the off-surface
targets).  Default workload: BASELINE.json configs[4] ("cfg5": 10,000 unit
spheres, p = 6, 980,000 nodes, 1,000,000 off-surface targets), the largest
configuration that exercises all rows; --config 4 times the 1.38M-node apply.

Metric (BASELINE.json): fp64 pair-interactions/s.  A pair is one (target,
source node) interaction of the fused SL+DL kernel: N (N - n_s) for the apply
(own sphere excluded) plus M N off-surface.  Inputs are resident in HBM when
the timed region starts; L2 (126 MB) is flushed between timed steps with a
256 MB write.  `e2e` times the host-buffer C-ABI entry points (pinned host
memory, H2D + D2H inside the timed region).

Multi-GPU: replicas only: each rank runs the same workload on
its own GPU, no data-path collective; value = total pairs / max-over-ranks time.

--impl reference times the CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same workload on the host cores.
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
sys.path.insert(0, ROOT)

# Algorithmic work per pair: 18 DFMA + 10 DMUL + 3 DADD = 31 FP64
# operations = 49 flops (FMA = 2) for the fused SL+DL pair; the off-surface
# pair with pressure adds 1 DADD + 1 DFMA = 33 operations = 52 flops.  (The
# kernel itself issues 30 / 32: DESIGN.md §5.)
FLOPS_PER_PAIR = 49
FLOPS_PER_PAIR_OFF = 52
FP64_OPS_PER_PAIR = 30   # FP64-pipe instructions the kernel issues per pair (apply)
FP64_OPS_PER_PAIR_OFF = 32
N_SM = 148
FP64_LANES = 64          # FP64 FMA lanes per SM (B200)
SM_MAX_MHZ = 1965.0
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")


def _hbm_peak_gbps():
    """Measured HBM copy bandwidth from MEASURED_PEAKS.json (driver-written);
    fallback when the file is absent: B200_PROFILING.md's 6650 GB/s."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


HBM_PEAK_GBPS = _hbm_peak_gbps()


def peak_fp64_tflops(mhz=SM_MAX_MHZ):
    """Derived FP64 FMA peak (guide unit counts x clock): context only."""
    return N_SM * FP64_LANES * 2 * mhz * 1e6 / 1e12


def measured_fp64_peak():
    """Measured FP64 CUDA-core peak (tools/fp64_peak.cu on a B200 of this pool,
    profiles/r02_fp64_peak.json): the best DFMA form, in TFLOP/s (FMA = 2), and
    the FP64 operations per SM per clock it sustained at its in-kernel clock.
    Returns (tflops, ops_per_sm_per_clk, source)."""
    try:
        best = None
        with open(FP64_PEAK_FILE) as fh:
            for line in fh:
                line = line.strip()
                if not line.startswith("{"):
                    continue
                r = json.loads(line)
                if r.get("op", "").startswith("DFMA") and (best is None or r["tflops"] > best["tflops"]):
                    best = r
        if best:
            return (float(best["tflops"]), float(best["ops_per_sm_per_clk"]),
                    f"measured: tools/fp64_peak.cu {best['op']} "
                    f"({os.path.relpath(FP64_PEAK_FILE, ROOT)}), {best['ops_per_s']:.4e} DFMA/s "
                    f"at {best['sm_mhz_in_kernel']:.0f} MHz in-kernel")
    except (OSError, KeyError, ValueError):
        pass
    return (peak_fp64_tflops(), float(FP64_LANES),
            "fallback (no measured file): 148 SM x 64 FP64 lanes x 2 x 1.965 GHz")


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank float over all ranks (torch.distributed; identity at world 1)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(pairs_per_step: int, steps: int, world: int, max_total_ms: float) -> float:
    """Whole-job throughput of N replicas: all ranks' pairs / max-over-ranks time."""
    return world * pairs_per_step * steps / (max_total_ms / 1e3)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def workload(cfg):
    from bie_inputs import make_config
    d = make_config(cfg, with_targets=(cfg == 5))
    return d


def nsn_of(p):
    return (p + 1) * (2 * p + 2)


def pair_counts(d):
    N = d["n_nodes"]
    ns = nsn_of(d["p"])
    apply_pairs = N * (N - ns)
    M = 0 if d["targets"] is None else len(d["targets"])
    return apply_pairs, M * N, M


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import torch
    import __graft_entry__
    __graft_entry__.build()  # no-op when libbie.so is up to date
    import paper_1707_06551_b200 as bie
    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    d = workload(args.config)
    from bie_inputs import rigid_field
    p, mu = d["p"], d["mu"]
    ctx = bie.bie_create(d["centres"], d["radii"], p, mu)
    N = bie.bie_num_nodes(ctx)
    f_np, q_np = d["f"], d["q"]
    if d["rigid"] is not None:
        x = torch.empty((N, 3), dtype=torch.float64, device=dev)
        bie.bie_get_nodes(ctx, x)
        q_np = rigid_field(*d["rigid"], x.cpu().numpy(), d["centres"], nsn_of(p))
    if d["same_fq"]:
        f_np = q_np
    f = torch.from_numpy(np.ascontiguousarray(f_np)).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(q_np)).to(dev)
    u = torch.empty((N, 3), dtype=torch.float64, device=dev)
    has_off = d["targets"] is not None
    if has_off:
        tg = torch.from_numpy(d["targets"]).to(dev)
        M = tg.shape[0]
        uo = torch.empty((M, 3), dtype=torch.float64, device=dev)
        po = torch.empty(M, dtype=torch.float64, device=dev)
    apply_pairs, off_pairs, M = pair_counts(d)
    step_pairs = apply_pairs + off_pairs
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        bie.bie_apply_SLDL(ctx, f, q, u, stream)
        if ev:
            ev[1].record(stream)
        if has_off:
            bie.bie_eval_offsurface(ctx, f, q, tg, uo, po, stream)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs)
    bie.bie_reset_profile(ctx)
    bie.bie_set_profiling(ctx, True)
    clocks = ClockSampler(local_rank)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    times, apply_times, off_times = [], [], []
    for _ in range(args.steps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        step(ev)
        ev[2].synchronize()
        times.append(ev[0].elapsed_time(ev[2]))
        apply_times.append(ev[0].elapsed_time(ev[1]))
        off_times.append(ev[1].elapsed_time(ev[2]))
    torch.cuda.synchronize()
    clk = clocks.stop()
    prof = bie.bie_get_profile(ctx)
    bie.bie_set_profiling(ctx, False)
    total_ms = max_over_ranks(sum(times), world, dev)
    apply_ms = max_over_ranks(sum(apply_times), world, dev)
    off_total_ms = max_over_ranks(sum(off_times), world, dev)
    ms_per_step = total_ms / args.steps
    # Headline: apply pairs / wall time of bie_apply_SLDL (pack +
    # self term + far field), CUDA events on the launching stream.  The
    # off-surface leg of the same step is reported separately ("offsurface").
    value = replica_value(apply_pairs, args.steps, world, apply_ms)
    launches = int(sum(v[1] for k, v in prof.items() if k != "copy"))

    peak, peak_ops_clk, peak_src = measured_fp64_peak()
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic_all = json.load(fh)
    except Exception:
        traffic_all = {}

    def kernel_roofline(kind, pairs, flops_per_pair, ops_per_pair, kname, rec_bytes, tgt_bytes,
                        traffic_key):
        ms = prof[kind][0] / args.steps  # ABI's CUDA events on the launching stream
        pairs_s = pairs / (ms / 1e3)
        achieved = pairs_s * flops_per_pair / 1e12
        tr = traffic_all.get(traffic_key)
        r = {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
             "frac": round(achieved / peak, 4),
             "traffic": (tr["dram_bytes_read"] + tr["dram_bytes_write"]) if tr else None,
             "algorithmic_bytes": rec_bytes + tgt_bytes,
             "traffic_source": (tr or {}).get("source"),
             "kernel": kname, "ms_per_launch_avg": round(ms / max(prof[kind][1] / args.steps, 1), 4),
             "ms_per_pass": round(ms, 4), "launches_per_pass": prof[kind][1] / args.steps,
             "pairs_per_s": pairs_s, "flops_per_pair": flops_per_pair,
             "peak_source": peak_src + " (of measured)",
             "fp64_pipe_frac_at_max_clock": round(pairs_s * ops_per_pair /
                                                  (N_SM * FP64_LANES * SM_MAX_MHZ * 1e6), 4)}
        if clk.get("sm_mhz"):
            r["fp64_pipe_frac_at_measured_clock"] = round(
                pairs_s * ops_per_pair / (N_SM * FP64_LANES * clk["sm_mhz"] * 1e6), 4)
        return r

    # dominant kernel of the headline: the apply's far-field pair sum (k_nbody)
    # Large launches (cfg 4, 5) run the constant-bank schedule: one far-field pass =
    # one launch of k_nbody_c per batch of 312 sources, alternating between two
    # streams (their launches overlap), plus the join; the pass is timed as a whole
    # by the ABI's events on the launching stream, and "achieved" = the pass's
    # algorithmic flops / that time (ms_per_pass; ms_per_launch_avg = pass time /
    # launches, the effective time per launch).
    const_a = prof["nbody"][1] / args.steps > 8
    roofline = kernel_roofline("nbody", apply_pairs, FLOPS_PER_PAIR, FP64_OPS_PER_PAIR,
                               "k_nbody_c<8,64,4,{0,1},false> (far-field SL+DL, row a3; sources as "
                               "constant-bank operands, batches of 312 over two streams)" if const_a else
                               "k_nbody<8,64,64,3,false> (far-field SL+DL, row a3)",
                               96 * N, 24 * N, f"cfg{args.config}_const" if const_a else f"cfg{args.config}")
    kernels = {k: {"ms_per_step": round(v[0] / args.steps, 4), "launches_per_step": v[1] / args.steps}
               for k, v in prof.items() if v[1]}
    offsurface = None
    if has_off and prof["offsurface"][0] > 0:
        const_o = prof["offsurface"][1] / args.steps > 8
        roff = kernel_roofline("offsurface", off_pairs, FLOPS_PER_PAIR_OFF, FP64_OPS_PER_PAIR_OFF,
                               "k_nbody_c<8,64,2,{0,1},true> (off-surface u and p, row a7; constant-bank "
                               "batches)" if const_o else "k_nbody<7,64,64,3,true> (off-surface u and p, row a7)",
                               104 * N, 32 * M, f"cfg{args.config}_off_const" if const_o else f"cfg{args.config}_off")
        offsurface = {"metric": "fp64 pair-interactions/sec, off-surface velocity + pressure (row a7)",
                      "value": replica_value(off_pairs, args.steps, world, off_total_ms),
                      "unit": "pair-interactions/s", "pairs_per_step": int(off_pairs),
                      "n_targets": int(M), "ms_per_step": off_total_ms / args.steps,
                      "roofline": roff}
    kernels["nbody"]["pairs_per_s"] = roofline["pairs_per_s"]
    if "self" in kernels and prof["self"][0] > 0:  # SHT stages (rows a2, a4-a6): HBM-bound by design
        self_s = prof["self"][0] / args.steps / 1e3
        self_bytes = 168 * N  # f, q in (48 B/node); records (96 B) + u (24 B) out
        kernels["self"]["algorithmic_bytes"] = self_bytes
        kernels["self"]["hbm_GBps"] = round(self_bytes / self_s / 1e9, 1)
        kernels["self"]["hbm_frac"] = round(self_bytes / self_s / 1e9 / HBM_PEAK_GBPS, 4)

    # ---- e2e through the host-buffer entry points (pinned host memory)
    e2e = None
    if not args.no_e2e:
        fh = torch.from_numpy(np.ascontiguousarray(f_np)).pin_memory()
        qh = torch.from_numpy(np.ascontiguousarray(q_np)).pin_memory()
        uh = torch.empty((N, 3), dtype=torch.float64).pin_memory()
        h2d = 2 * N * 3 * 8   # f, q
        d2h = N * 3 * 8       # u
        if has_off:
            tgh = torch.from_numpy(d["targets"]).pin_memory()
            uoh = torch.empty((M, 3), dtype=torch.float64).pin_memory()
            poh = torch.empty(M, dtype=torch.float64).pin_memory()
            h2d_off = 2 * N * 3 * 8 + M * 3 * 8
            d2h_off = M * 4 * 8

        def step_host(ev=None):
            if ev:
                ev[0].record(stream)
            bie.bie_apply_SLDL_host(ctx, fh, qh, uh, stream)
            if ev:
                ev[1].record(stream)
            if has_off:
                bie.bie_eval_offsurface_host(ctx, fh, qh, tgh, uoh, poh, stream)
            if ev:
                ev[2].record(stream)

        step_host()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ea, eo = [], []
        for _ in range(args.e2e_steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            step_host(ev)
            ev[2].synchronize()
            ea.append(ev[0].elapsed_time(ev[1]))
            eo.append(ev[1].elapsed_time(ev[2]))
        tot_a = max_over_ranks(sum(ea), world, dev)
        e2e = {"value": replica_value(apply_pairs, args.e2e_steps, world, tot_a), "unit": "pair-interactions/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "ms_per_step": tot_a / args.e2e_steps,
               "note": "apply pairs / time of bie_apply_SLDL_host (pinned host f, q in; u out; "
                       "H2D + D2H inside the timed region)"}
        if has_off and offsurface is not None:
            tot_o = max_over_ranks(sum(eo), world, dev)
            offsurface["e2e"] = {"value": replica_value(off_pairs, args.e2e_steps, world, tot_o),
                                 "unit": "pair-interactions/s", "h2d_bytes_per_step": h2d_off,
                                 "d2h_bytes_per_step": d2h_off, "ms_per_step": tot_o / args.e2e_steps,
                                 "note": "bie_eval_offsurface_host (f, q, targets in; u, p out)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(d, f_np, q_np, budget_s=args.cpu_seconds)

    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    if rank != 0:
        return
    cfg_names = {4: "cfg4: 4096 unit spheres jittered lattice, p=12, D[q]+S[q]",
                 5: "cfg5: 10000 unit spheres RSA side 60, p=6, apply + 1e6 off-surface targets"}
    out = {
        "metric": "fp64 pair-interactions/sec for SL+DL apply; % of B200 FP64 peak",
        "value": value, "unit": "pair-interactions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "apply_ms_per_step": apply_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json recipe, bie_inputs/)",
        "config": {"workload": f"cfg{args.config}",
                   "description": cfg_names.get(args.config, CONFIG_DESC(args.config)),
                   "n_spheres": int(len(d["radii"])), "p": p, "n_nodes": int(N),
                   "n_offsurface_targets": int(M), "apply_pairs": int(apply_pairs),
                   "offsurface_pairs": int(off_pairs), "l2": "flushed (256 MB write) between timed steps",
                   "value_is": "apply pairs / bie_apply_SLDL wall time (SURVEY §8(d)); "
                               "ms_per_step is the whole step (apply + off-surface)",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "roofline": roofline,
        "offsurface": offsurface,
        "step_value": replica_value(step_pairs, args.steps, world, total_ms),
        "step_value_note": "all pairs of the step (apply + off-surface) / whole-step time",
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk,
        "gpu_launches": launches,
        "kernels": kernels,
        "step_ms": [round(t, 3) for t in times],
    }
    print(json.dumps(out))


def CONFIG_DESC(c):
    from bie_inputs import CONFIGS
    return CONFIGS.get(c, "")


# ------------------------------------------------------------------ CPU oracle
def cpu_baseline(d, f_np, q_np, budget_s=15.0, kind="oracle", legs=("apply",)):
    """Time the oracle (as it stands) on a bounded random sample of the workload:
    batches of random target nodes of the apply (far field + self term; and,
    with legs including "off", off-surface targets) are evaluated until the time
    budget is spent; value = pairs evaluated / wall time (the headline metric's
    unit: apply pairs/s)."""
    import oracle
    oracle.build_oracle()
    cores = oracle.num_threads()
    N = d["n_nodes"]
    ns = nsn_of(d["p"])
    rng = np.random.default_rng(12345)
    has_off = d["targets"] is not None and "off" in legs
    legs = [("apply", N - ns, N)] + ([("off", N, len(d["targets"]))] if has_off else [])
    share = budget_s / len(legs)
    tot_t, tot_p, desc = 0.0, 0, []
    for leg, pairs_per_target, pool in legs:
        t_leg, n_leg, batch = 0.0, 0, max(8, 2 * cores)
        while t_leg < share and n_leg < pool:
            nt = int(min(batch, pool - n_leg))
            t0 = time.perf_counter()
            if leg == "apply":
                sub = np.sort(rng.choice(N, nt, replace=False))
                oracle.apply(d["centres"], d["radii"], d["p"], d["mu"], f_np, q_np, sub)
            else:
                idx = np.sort(rng.choice(pool, nt, replace=False))
                oracle.offsurface(d["centres"], d["radii"], d["p"], d["mu"], f_np, q_np,
                                  d["targets"][idx])
            dt = time.perf_counter() - t0
            t_leg += dt
            n_leg += nt
            rate = nt / max(dt, 1e-6)
            batch = max(8, int(rate * (share - t_leg) * 1.05))
        tot_t += t_leg
        tot_p += n_leg * pairs_per_target
        desc.append(f"{n_leg} random {'nodes of the apply (far + self)' if leg == 'apply' else 'off-surface targets'}")
    return {"value": tot_p / tot_t, "unit": "pair-interactions/s", "cores": cores, "kind": kind,
            "sample": " + ".join(desc) + f" of cfg{d['cfg']}, {tot_t:.1f} s wall"}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    d = workload(args.config)
    f_np, q_np = d["f"], d["q"]
    if d["rigid"] is not None:
        import oracle
        x, _, _ = oracle.nodes(d["centres"], d["radii"], d["p"])
        from bie_inputs import rigid_field
        q_np = rigid_field(*d["rigid"], x, d["centres"], nsn_of(d["p"]))
    if d["same_fq"]:
        f_np = q_np
    per_step = max(2.0, args.cpu_seconds / max(args.steps, 1))
    for _ in range(args.warmup):
        cpu_baseline(d, f_np, q_np, budget_s=0.2)
    vals, secs = [], 0.0
    res = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = cpu_baseline(d, f_np, q_np, budget_s=per_step)
        secs += time.perf_counter() - t0
        vals.append(res["value"])
    v = float(np.median(vals))
    res["value"] = v
    out = {"impl": "reference", "metric": "fp64 pair-interactions/sec for SL+DL apply; % of B200 FP64 peak",
           "value": v, "unit": "pair-interactions/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded BASELINE.json recipe, bie_inputs/)",
           "config": {"workload": f"cfg{args.config}", "note": "CPU oracle on a bounded sample per step"},
           "cpu_baseline": res,
           "e2e": {"value": v, "unit": "pair-interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[2, 3, 4, 5])
    ap.add_argument("--impl", default="bie", choices=["bie", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=30.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: RREF + transformation over GF(q) (arXiv 1806.04211 Chief) on B200.

One step = one full ``echelonize`` (ChopMatrix -> Steps 1-3 -> EchelonOutput,
with transformation) of the largest BASELINE.json configuration that fits one
GPU: configs[4]'s 1-GPU case, GF(2) 65536 x 65536, iid uniform entries
(reference random_matrix, seed 1, generated on the device by K6), block 8192
(an 8 x 8 block grid).  ``--config`` selects the other configs.
Metric: effective GF(q) mult-adds/s = m*n*r / step time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  Multi-GPU (N > 1, torchrun, one process
per GPU): the same job runs as the block-column sharded Chief (block
columns round-robin over the ranks, PkgA / X packages broadcast over NCCL),
so the scaling is strong (fixed total work).
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

from paper_1806_04211_b200.workloads import CONFIGS  # noqa: E402

DEFAULT = "cfg5s"
METRIC = "RREF+transform effective GF(q) mult-adds/s (m*n*r / wall)"
UNIT = "mult-adds/s"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def setup_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    return world, rank, local, dist


def ref_sample(cfg):
    """The reference's CPU sample of a workload: the leading s x s submatrix
    with the config's block GRID kept (block = s / grid), so the reference
    runs the same Chief task DAG as the full job, scaled.  s = the full size
    when it is at most 8192 (cfg1 / cfg2a: the exact config), else 8192:
    at cfg5s's own block (8192) any sample that bounded is ONE block, which
    the reference would eliminate in a single task on one thread."""
    grid = max(1, cfg["m"] // cfg["block"])
    side = min(cfg["m"], cfg["n"])
    if side <= 8192:
        s = side
        blk = cfg["block"]
    else:
        s = 8192 // grid * grid
        blk = s // grid
    same = s == cfg["m"] and s == cfg["n"] and blk == cfg["block"]
    label = (f"full {cfg['m']}x{cfg['n']} input, block {blk}" if same else
             f"leading {s}x{s} of the {cfg['m']}x{cfg['n']} input, block {blk} (the config's "
             f"{grid}x{grid} block grid, scaled: the full job does not fit host RAM / minutes)")
    return s, blk, same, label


def cpu_baseline(cfg, C):
    """The reference library (oracle/_ref, compiled from /root/reference) on
    the host cores, all threads, once, on ref_sample's bounded sample."""
    import oracle
    if oracle.ref is None:
        return None
    threads = max(1, oracle.ref.ref_hardware_concurrency())
    s, blk, same, label = ref_sample(cfg)
    if cfg["kind"] == "random":   # the leading rows of the same row-major draw stream
        sample = oracle.random_matrix(cfg["p"], s, cfg["n"], cfg["seed"])[:, :s].copy()
    else:
        sample = C.numpy()[:s, :s].copy()
    t0 = time.time()
    o = oracle.ref_echelonize(cfg["p"], sample, blk, threads=threads)
    wall = time.time() - t0
    work = s * s * o.rank
    return {"value": work / wall, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{label}; gfrref::echelonize with_transform, {threads} threads, 1 call, {wall:.2f} s",
            "same_config": same, "wall_s": wall}


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref)
    with all host threads; each step one call on ref_sample's sample."""
    if rank != 0:
        return
    import oracle
    if oracle.ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgfrref_ref.so not built"}))
        return
    threads = max(1, oracle.ref.ref_hardware_concurrency())
    if cfg["kind"] != "random":
        print(json.dumps({"impl": "reference", "unavailable": "reference arm wired for the random workloads only"}))
        return
    s, blk, same, label = ref_sample(cfg)
    # the leading s x s of random_matrix(m, n) (row-major draws): rows of the
    # full stream, generated by the reference itself only where they fit
    C = oracle.random_matrix(cfg["p"], s, cfg["n"], cfg["seed"]) if s < cfg["m"] else \
        oracle.random_matrix(cfg["p"], cfg["m"], cfg["n"], cfg["seed"])
    sample = C[:s, :s].copy()
    for _ in range(args.warmup):
        oracle.ref_echelonize(cfg["p"], sample, blk, threads=threads)
    walls, work = [], 0
    for _ in range(args.steps):
        t0 = time.time()
        o = oracle.ref_echelonize(cfg["p"], sample, blk, threads=threads)
        walls.append(time.time() - t0)
        work += s * s * o.rank
    tot = sum(walls)
    val = work / tot
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32 (reference Elem)",
            "data": "synthetic: reference random_matrix seed 1 (host)",
            "config": {"workload": cfg["desc"], "p": cfg["p"], "m": cfg["m"], "n": cfg["n"], "block": cfg["block"],
                       "sample": label, "sample_block": blk, "same_config": same},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{label}, per step"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def load_traffic(config):
    """Per-family DRAM traffic of one launch of the config's dominant shape
    (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum), from
    profiles/r02_traffic.json; {} when not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            return json.load(f).get(config, {})
    except Exception:
        return {}


def dominant_shape(config):
    """The K1 shape with the most work in one step of the config (GFQ_MAD_LOG)."""
    return {"cfg5s": (8192, 65536, 8192), "cfg4": (4096, 32768, 4096), "cfg3": (2048, 12288, 2048),
            "cfg2a": (1024, 8192, 1024), "cfg2b": (1024, 8192, 1024), "cfg1": (500, 2000, 500)}.get(config)


def k1_isolated(G, p, peak, dominant=None, policy=2):
    """K1 alone on a quiet device: CUDA events around back-to-back launches
    (after 3 warm-ups) through gfq_mad_raw on the current stream, tcgen05
    path forced (policy 2: kind::i8; 3: the FP4 path, its two operand
    packing passes included); shapes: the 1024^3 block product and the
    step's dominant shape."""
    import torch
    out = []
    shapes = [(1024, 1024, 1024)]
    if dominant and dominant not in shapes:
        shapes.append(dominant)
    G.set_mad_policy(policy)
    try:
        for (m, n, k) in shapes:
            A = torch.randint(0, p, (m, k), dtype=torch.uint8, device="cuda")
            Bm = torch.randint(0, p, (k, n), dtype=torch.uint8, device="cuda")
            D = torch.zeros((m, n), dtype=torch.uint8, device="cuda")
            G.set_stream(torch.cuda.current_stream().cuda_stream)
            call = lambda: G.mad_raw(p, m, n, k, A.data_ptr(), k, Bm.data_ptr(), n, D.data_ptr(), n,
                                     D.data_ptr(), n)
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            reps = 20 if m * n * k < 1 << 34 else 5
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            e1.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / reps
            tops = 2.0 * m * n * k / (us * 1e-6) / 1e12
            out.append({"shape": f"{m}x{n}x{k}", "us": us, "tflops": tops, "frac": tops / peak})
            del A, Bm, D
    finally:
        G.set_mad_policy(0)
        G.set_stream(0)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT, choices=sorted(CONFIGS))
    ap.add_argument("--threads", type=int, default=4, help="host workers / CUDA streams of the DAG executor")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world, rank, local, dist = setup_dist()
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    from paper_1806_04211_b200 import gfrref as G
    G.lib()
    f = G.FieldSpec(cfg["p"])
    from paper_1806_04211_b200 import workloads
    if cfg.get("sharded_only") and world < 4:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "unavailable": f"{args.config} ({cfg['m']}x{cfg['n']} u8 = "
                              f"{cfg['m'] * cfg['n'] / 2**30:.0f} GiB input) runs sharded over >= 4 GPUs only"}))
        if dist:
            dist.destroy_process_group()
        return
    # the full-size cfg5 never exists on one GPU: every rank generates only
    # its own block columns of the seeded stream (K6) inside the call
    C = None if cfg.get("sharded_only") else workloads.build(G, args.config)
    opts = G.EchelonizeOptions(block=cfg["block"], threads=args.threads, with_transform=True)
    # the one-time mapping of the device pool (cfg5s: ~3.5 s) before any step
    # (sharded: this rank's share of the block columns)
    G.reserve_for(cfg["m"], max(1, cfg["n"] // world), True)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # N > 1: the block-column sharded Chief over NCCL, one
    # process per GPU; block columns round-robin, PkgA / X broadcasts.
    comm = None
    if world > 1:
        ids = [G.Comm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        comm = G.Comm.nccl(world, rank, ids[0])

    def step(Cin=None, gather=False):
        Cin = C if Cin is None else Cin
        if comm is not None:
            return G.echelonize_dist(comm, f, cfg["m"], cfg["n"], opts, C=Cin, seed=cfg["seed"], gather=gather)
        return G.echelonize(Cin, f, opts)

    rank_r = step(gather=True).rank
    for _ in range(max(args.warmup, 0)):
        out = step()
        del out
    work = cfg["m"] * cfg["n"] * rank_r

    # ---------------- timed region (device-resident input)
    G.launch_count(reset=True)
    G.device_memory(reset_peak=True)
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    times, walls = [], []
    for _ in range(args.steps):
        flush.fill_(1)  # > L2 (126 MB): evict between steps, outside the events
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record()
        out = step()
        e1.record()
        e1.synchronize()
        walls.append(time.perf_counter() - h0)
        times.append(e0.elapsed_time(e1))
        del out
    barrier()
    clk = clocks.stop()
    launches = G.launch_count(reset=True)
    dm = G.device_memory()
    if dist:
        t = torch.tensor([float(dm["peak"])], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dm["peak"] = int(t.item())
    hbm = {"high_water_bytes": dm["peak"], "input_bytes": cfg["m"] * cfg["n"],
           "high_water_over_input": dm["peak"] / (cfg["m"] * cfg["n"]),
           "pool_reserved_high_bytes": dm["pool_reserved_high"],
           "note": "the library's device allocations (matrices, panels, scratch) during the timed steps, "
                   "max over ranks; the input and one step's outputs included"}
    # K1 per-launch device timing: the same steps again with CUDA events
    # around every K1 launch on its worker stream (kept out of the timed
    # region above: the events add host work per launch).
    G.profile(True)
    G.profile_take_kinds()
    prof_ms = []
    for _ in range(args.steps):
        flush.fill_(3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = step()
        e1.record()
        e1.synchronize()
        prof_ms.append(e0.elapsed_time(e1))
        del out
    prof = G.profile_take_kinds(with_union=True)
    G.profile(False)
    tot_ms = sum(times)
    if dist:
        t = torch.tensor([tot_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    # strong scaling: the same job sharded over the N GPUs
    value = work * args.steps / (tot_ms / 1e3)

    # ---------------- e2e: public API with host buffers (H2D + D2H inside)
    e2e = None
    if cfg.get("sharded_only") and not args.no_e2e:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": f"{args.config}'s {cfg['m'] * cfg['n'] / 2**30:.0f} GiB input has no host copy: each rank "
                       "generates its own block columns on the device"}
    elif not args.no_e2e:
        Ch = torch.empty((cfg["m"], cfg["n"]), dtype=torch.uint8, pin_memory=True)
        Ch.numpy()[:] = C.numpy()
        probe = step(gather=True)
        nbytes = probe.block_bytes()
        del probe
        dl = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        barrier()
        et = []
        for _ in range(max(1, min(args.steps, 5))):
            flush.fill_(2)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if comm is None:
                # H2D inside the call; every output block streams into the
                # pinned `dl` as soon as it is final (D2H overlaps Step 3)
                out = G.echelonize(Ch.numpy(), f, opts, host_out=dl.numpy())
            else:
                out = step(Cin=G.Matrix.from_numpy(Ch.numpy()), gather=True)
                if rank == 0:
                    out.download_blocks(dl.numpy())
            sel_bytes = 4 * out.rank * 2
            if comm is None:
                xfer = G.last_transfer_bytes()  # what crossed PCIe inside the call
            e1.record()
            e1.synchronize()
            et.append(e0.elapsed_time(e1))
            del out
        e_ms = sum(et) / len(et)
        if dist:
            t = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": work / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": xfer[0] if comm is None else world * cfg["m"] * cfg["n"],
               "d2h_bytes_per_step": int((xfer[1] if comm is None else nbytes) + sel_bytes), "ms_per_step": e_ms,
               "path": "gfq_echelonize_host_into (pinned host C -> HBM, every output block -> pinned host as it becomes final)" if comm is None
               else "each rank uploads pinned host C, gfq_echelonize_dist(gather), rank 0 downloads all blocks"}

    # ---------------- rooflines of the two kernel families with the most device time
    peaks = measured_peaks()
    if peaks and peaks.get("bf16_tflops"):
        tpeak = 2.0 * peaks["bf16_tflops"]
        tpeak_src = "2 x measured cuBLAS bf16 burst (MEASURED_PEAKS.json); B200 dense int8 = 2 x dense bf16"
    else:
        tpeak = 2.0 * 1590.0
        tpeak_src = "fallback 2 x 1.59 PF bf16 (B200_PROFILING.md)"
    if peaks and peaks.get("hbm_gbs"):
        hpeak, hpeak_src = peaks["hbm_gbs"], "measured copy bandwidth (MEASURED_PEAKS.json)"
    else:
        hpeak, hpeak_src = 7672.0, "fallback (B200_PROFILING.md)"
    # the FP4 path (kind::mxf4) peaks at 4 x dense bf16 (B200: 9 vs 2.25 PF nominal)
    f4peak = 2.0 * tpeak
    f4peak_src = tpeak_src.replace("2 x measured", "4 x measured").replace(
        "B200 dense int8 = 2 x dense bf16", "B200 dense fp4 = 4 x dense bf16")
    names = {"k1_tc": "gf_mad_tc_kernel (K1, tcgen05.mma kind::i8)",
             "k1_f4": "gf_mad_f4_kernel (K1f, tcgen05.mma kind::mxf4, E2M1 residues, fp32 sums)",
             "k1_simt": "mad_smallk / mad_simt (K1 SIMT, K < 32)",
             "ech_gf2": "ech_gf2_cluster_kernel (K2, GF(2) 8-CTA cluster ECH)",
             "ech_panel": "ech_step_chain / ech_step_update / ech_panel (K2, general p)",
             "select": "select2d_v16 / select_rows_v16 / select_inline (K3/K4 gathers, riffles) + "
                       "pack_rows_f4 / pack_cols_f4 (K1f operand packing)"}
    traffic = load_traffic(args.config)
    step_ms = sum(prof_ms) / max(1, len(prof_ms))
    roofs = []
    for fam, (nl, wk, ms, ums) in sorted(prof.items(), key=lambda kv: -kv[1][3]):
        if nl == 0 or ums <= 0:
            continue
        tensor = fam.startswith("k1")
        ach = wk / (ums / 1e3) / (1e12 if tensor else 1e9)
        peak = (f4peak if fam == "k1_f4" else tpeak) if tensor else hpeak
        tr = traffic.get(fam)
        nsteps = max(1, args.steps)
        roofs.append({"kernel": names.get(fam, fam), "family": fam, "bound": "tensor" if tensor else "hbm",
                      "achieved": ach, "peak": peak, "unit": "TFLOP/s" if tensor else "GB/s",
                      "frac": ach / peak, "traffic": tr["dram_bytes"] if tr else None,
                      "traffic_shape": tr["shape"] if tr else None,
                      "traffic_algorithmic": tr["algorithmic_bytes"] if tr else None,
                      "peak_source": (f4peak_src if fam == "k1_f4" else tpeak_src) if tensor else hpeak_src,
                      "work_per_launch": wk / nl, "work_unit": "int8 ops (2 x MACs)" if tensor else
                      "algorithmic bytes (u8 payload read + written, +4 B per index)",
                      "launches_per_step": nl / nsteps, "avg_launch_us": 1e3 * ms / nl,
                      "busy_ms_per_step": ums / nsteps, "event_ms_per_step": ms / nsteps,
                      "share_of_step": ums / nsteps / step_ms if step_ms else None})
        if len(roofs) == 2:
            break
    note = ("achieved = the family's algorithmic work / its busy time: CUDA events around every launch "
            f"on its worker stream over {args.steps} profiled steps run right after the timed region "
            f"({step_ms:.2f} ms/step with events), the launch windows merged on one device clock so "
            "concurrent launches on several streams count once (they still share SMs with the other "
            "families); event_ms_per_step = the unmerged sum; traffic = ncu dram__bytes_read+write of one "
            "launch of the step's dominant shape run alone (profiles/r02_traffic.json)")
    roof = dict(roofs[0]) if roofs else {}
    roof["note"] = note
    roof["second"] = roofs[1] if len(roofs) > 1 else None
    roof["families"] = {k: {"launches": v[0], "work": v[1], "event_ms": v[2], "busy_ms": v[3]}
                        for k, v in prof.items()}

    # K1 timed alone (no concurrent streams), CUDA events around back-to-back
    # launches: the block product and the step's dominant shape
    if rank == 0:
        roof["isolated"] = k1_isolated(G, cfg["p"], tpeak, dominant_shape(args.config))
        if cfg["p"] in (2, 3, 5, 7):
            roof["isolated_f4"] = k1_isolated(G, cfg["p"], f4peak, dominant_shape(args.config), policy=3)

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(cfg, C)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u8",
                "data": f"synthetic: {cfg['kind']} GF({cfg['p']}) input, seed {cfg['seed']}, generated on the "
                        f"device by K6/K1 (bit-identical to the reference generators; workloads.py)",
                "config": {"workload": cfg["desc"], "p": cfg["p"], "m": cfg["m"], "n": cfg["n"],
                           "block": cfg["block"], "rank": rank_r, "with_transform": True,
                           "executor_streams": args.threads,
                           "l2": "flushed (512 MiB device write) before every timed step",
                           "parallelism": f"block-column sharded Chief over {world} GPUs (NCCL broadcasts)"
                           if world > 1 else "1 GPU"},
                "wall_ms_per_step": 1e3 * sum(walls) / len(walls),
                "roofline": roof, "cpu_baseline": base, "e2e": e2e, "clocks": clk,
                "hbm": hbm,
                "gpu_launches": launches}
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Benchmark: GCUPS of the B200 inter-task Smith-Waterman search
(BASELINE.json metric) on BASELINE.json configs[1] -- a query of 464 residues
against 1,000,000 synthetic sequences (~200 M residues), one B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one pass of the whole hot path over the resident database
(SURVEY.md 8(a) rows a2-a6): query-profile build, the s16x2 pass kernel(s),
saturation flag compaction + exact s32 re-scoring, and the sorting stage
(device top-10).  Pre-processing (sw_db_load, row a1) is done once before the
timed region, as in the paper.  GCUPS = |Q||D| /
(t 1e9) (Eq. 4).  N > 1 (torchrun): weak scaling -- the database
is configs[1] x N, residue-balanced over the ranks, each rank searches its
shard and the per-rank scores and top-10 are gathered to rank 0 over NCCL and
merged there.  Rank 0 prints one JSON line.
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

import sw_inputs as si  # noqa: E402

METRIC = "GCUPS (giga cell updates/sec) at 1/2/4/8 B200, % of int/DPX roofline"
CONFIG_INDEX = 1
TOPK = 10
ALU_LANE_OPS_PER_CLK_PER_SM = 64      # measured (profiles/r01_dpx_microbench.jsonl); guide: rt_SMSP=2
# ALU-pipe instructions per cell of the 16-bit pass kernel:
# biased arithmetic 4.5 per s16x2 pair of cells (VIMNMX3 + 3 VIADDMNMX + 1/2
# VIMNMX3; the diagonal add runs on the FMA pipe), relu form 5.5 DPX.
ALU_PER_CELL = {1: 2.25, 0: 2.75}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG_INDEX)
    ap.add_argument("--scale", type=float, default=1.0, help="(dev) shrink the workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="initialise the NCCL process group even at world size 1 (exercises the gather path)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [x for x in sm if x > 500] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    return {"sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md nominal clocks)"


def ncu_pipes():
    """ALU-pipe thread instructions per cell of the pass kernel, measured by ncu
    on the bench launch (profiles/r01b_ncu_pipes.json), for the roofline with
    the kernel's measured I_pipe."""
    p = os.path.join(ROOT, "profiles", "r01b_ncu_pipes.json")
    try:
        with open(p) as f:
            return json.load(f).get("alu_thread_inst_per_cell")
    except Exception:
        return None


def ncu_traffic():
    """DRAM bytes per launch of the pass kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                d = json.load(f)
            return d.get("sw16_dram_bytes_per_launch")
        except Exception:
            return None
    return None


def cpu_baseline(w, target_s: float = 12.0):
    """The oracle (oracle/, plain scalar C, one sequence per task on all host
    cores) timed on a bounded seeded sample of the same workload."""
    import oracle
    q = w.queries[0]
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(7195)
    perm = rng.permutation(w.db.count)
    lens = w.db.lengths()
    # calibrate on a small sample, then size the sample for ~target_s seconds
    cal = perm[:2000]
    t0 = time.perf_counter()
    oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend, idx=cal, threads=cores)
    dt = max(time.perf_counter() - t0, 1e-3)
    rate = len(q) * int(lens[cal].sum()) / dt
    want_res = target_s * rate / len(q)
    csum = np.cumsum(lens[perm])
    nsamp = int(min(w.db.count, max(2000, np.searchsorted(csum, want_res))))
    idx = perm[:nsamp]
    t0 = time.perf_counter()
    oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend, idx=idx, threads=cores)
    dt = time.perf_counter() - t0
    cells = len(q) * int(lens[idx].sum())
    return {"value": round(cells / dt / 1e9, 3), "unit": "GCUPS", "cores": cores, "kind": "oracle",
            "sample": f"{nsamp} seeded-random sequences of the workload ({int(lens[idx].sum())} residues) "
                      f"vs the {len(q)}-residue query, {dt:.1f} s"}


def make_workload(args, world):
    scale = args.scale * (world if world > 1 else 1)
    return si.make_config(args.config, scale=scale)


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    w = make_workload(args, world)
    q = w.queries[0]
    cores = os.cpu_count() or 1
    lens = w.db.lengths()
    rng = np.random.default_rng(1702)
    perm = rng.permutation(w.db.count)
    # size each step's sample so warmup+steps finish in ~2-3 minutes
    budget = max(2.0, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    cal = perm[:1000]
    t0 = time.perf_counter()
    oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend, idx=cal, threads=cores)
    rate = len(q) * int(lens[cal].sum()) / max(time.perf_counter() - t0, 1e-3)
    csum = np.cumsum(lens[perm])
    nsamp = int(min(w.db.count, max(1000, np.searchsorted(csum, budget * rate / len(q)))))
    times, cells = [], 0
    for s in range(args.warmup + args.steps):
        idx = perm[(s * nsamp) % max(1, w.db.count - nsamp):][:nsamp]
        t0 = time.perf_counter()
        sc = oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend, idx=idx,
                          threads=cores)
        oracle.topk(sc, TOPK)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            cells += len(q) * int(lens[idx].sum())
    total = sum(times)
    val = cells / total / 1e9
    sample = f"{nsamp} sequences per step (seeded, ~{budget:.0f} s each) of {w.name}, query {len(q)}"
    line = {"metric": METRIC, "value": round(val, 3), "unit": "GCUPS", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * total / max(1, len(times)), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "i64", "data": "synthetic",
            "config": {"workload": w.name, "query_len": len(q), "db_sequences": w.db.count,
                       "db_residues": w.db.total_residues},
            "cpu_baseline": {"value": round(val, 3), "unit": "GCUPS", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(val, 3), "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_1702_07195_b200 as sw
    from paper_1702_07195_b200 import build as swbuild
    from paper_1702_07195_b200.parallel import gather_to_root, shard_arrays, shard_database

    world, rank, local = dist_env()
    assert torch.cuda.is_available(), "bench needs a CUDA device"
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.dist:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        swbuild.build()
    if dist:
        dist.barrier()

    w = make_workload(args, world)
    q = w.queries[0]
    if world > 1:
        shards = shard_database(w.db.lengths(), world)
        gidx = shards[rank]
        res, offs = shard_arrays(w.db.residues, w.db.offsets, gidx)
    else:
        gidx = np.arange(w.db.count, dtype=np.int64)
        res, offs = w.db.residues, w.db.offsets
    count = int(offs.size - 1)
    local_res = int(offs[-1])
    sw.sw_db_load(res, offs)

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    d_scores = torch.empty(count, dtype=torch.int32, device=dev)
    d_gidx = torch.from_numpy(gidx.astype(np.int64)).to(dev)
    d_tk_i = torch.empty(TOPK, dtype=torch.int64, device=dev)
    d_tk_s = torch.empty(TOPK, dtype=torch.int32, device=dev)
    nmax = count
    if dist:
        t = torch.tensor([count], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nmax = int(t.item())
    d_pad = torch.zeros(nmax, dtype=torch.int32, device=dev)
    m_tk_i = torch.empty(TOPK, dtype=torch.int64, device=dev)
    m_tk_s = torch.empty(TOPK, dtype=torch.int32, device=dev)
    launches_per_step = [0]

    def step():
        sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d_scores, stream)
        sw.sw_topk_dev(d_scores, d_gidx, count, TOPK, d_tk_i, d_tk_s, stream)
        n = 0
        if dist:
            with torch.cuda.stream(stream):
                d_pad[:count].copy_(d_scores)
                all_sc = gather_to_root(d_pad, world, rank, dist)
                all_ti = gather_to_root(d_tk_i, world, rank, dist)
                all_ts = gather_to_root(d_tk_s, world, rank, dist)
                if rank == 0:
                    cand_i = torch.cat(all_ti)
                    cand_s = torch.cat(all_ts)
                    sw.sw_topk_dev(cand_s, cand_i, cand_s.numel(), TOPK, m_tk_i, m_tk_s, stream)
                    n += 3
                del all_sc
        return n

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    st = sw.sw_last_stats()
    # qp build, P x (pass kernel + score gather + flag compaction + s32 re-scoring
    # of that pass's newly flagged sequences), P-1 item-skip launches (between
    # passes), top-k (2 + decode)
    per_step_kernels = 1 + 4 * st["passes"] + max(0, st["passes"] - 1) + 3
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    extra = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        extra += step()
        kernel_ms.append(sw.sw_last_timing()["pass_kernels_ms"])
    e1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    total_res = w.db.total_residues
    gcups = len(q) * total_res / (ms_step * 1e6)

    # ---- end to end through the public C-ABI with host buffers (rank-local)
    e2e_val = None
    h2d = len(q) + 576
    d2h = count * 4 + TOPK * 12
    if True:
        import torch as _t
        host_scores = _t.empty(count, dtype=_t.int32, pin_memory=True).numpy()
        qpin = _t.empty(len(q), dtype=_t.uint8, pin_memory=True).numpy()
        qpin[:] = q
        mpin = _t.empty((24, 24), dtype=_t.int8, pin_memory=True).numpy()
        mpin[:] = w.matrix
        for _ in range(2):
            sw.sw_search(qpin, mpin, w.gap_open, w.gap_extend, out=host_scores)
            sw.sw_topk(TOPK)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        ne = max(3, args.steps // 3)
        for _ in range(ne):
            sw.sw_search(qpin, mpin, w.gap_open, w.gap_extend, out=host_scores)
            sw.sw_topk(TOPK)
        dt = (time.perf_counter() - t0) / ne
        if dist:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e_val = len(q) * total_res / (dt * 1e9)

    # ---- roofline of the dominant kernel (s16x2 pass kernel, ALU/DPX bound)
    peaks, peaks_src = measured_peaks()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    kms = float(np.mean(kernel_ms))
    achieved = len(q) * local_res / (kms * 1e6)          # GCUPS of the pass kernels, this rank
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    alu_per_cell = ALU_PER_CELL[int(sw.sw_last_stats()["arith"])]
    peak = nsm * f_max * 1e6 * ALU_LANE_OPS_PER_CLK_PER_SM / alu_per_cell / 1e9
    f_obs = clk.get("sm_mhz")
    roof = {"bound": "alu", "achieved": round(achieved, 1), "peak": round(peak, 1), "unit": "GCUPS",
            "frac": round(achieved / peak, 4), "traffic": ncu_traffic(),
            "kernel": "sw16_pass_kernel", "kernel_ms": round(kms, 4),
            "kernel_share_of_step": round(kms / ms_step, 4),
            "peak_basis": f"{nsm} SMs x {f_max:.0f} MHz (sm_max_mhz, {peaks_src}) x "
                          f"{ALU_LANE_OPS_PER_CLK_PER_SM} ALU lane-ops/clk/SM / {alu_per_cell} ALU instructions per cell",
            "frac_at_observed_clock": (round(achieved / (peak * f_obs / f_max), 4) if f_obs else None)}
    # SURVEY.md 8(d) D5's two other fractions: against the bound with the
    # kernel's measured ALU instructions per cell (ncu), and against the relu
    # form's 5.5 DPX per pair of cells (2.75 per cell)
    ipipe = ncu_pipes()
    if ipipe:
        roof["frac_measured_ipipe"] = round(achieved / (nsm * f_max * 1e6 * ALU_LANE_OPS_PER_CLK_PER_SM / ipipe / 1e9), 4)
        roof["ipipe_alu_per_cell"] = ipipe
    roof["frac_vs_2.75_dpx_per_cell"] = round(achieved / (nsm * f_max * 1e6 * ALU_LANE_OPS_PER_CLK_PER_SM / 2.75 / 1e9), 4)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gcups, 1), "unit": "GCUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i16",
            "data": "synthetic",
            "config": {"workload": f"{w.name}: query {len(q)} vs {w.db.count} synthetic sequences "
                                   f"({total_res} residues), BLOSUM62, gaps 10/2",
                       "query_len": len(q), "db_sequences": w.db.count, "db_residues": total_res,
                       "per_gpu_db_residues": local_res, "topk": TOPK,
                       "tile_G_R": [st["G"], st["R"]], "passes": st["passes"],
                       "flagged_rescored": st["flagged"],
                       "l2": "inputs larger than L2 (stream image %.0f MB > 126 MB)" % (st["pair_columns"] * 4 / 1e6),
                       "parallelism": f"dp{world} (database shards)"},
            "e2e": {"value": round(e2e_val, 1) if e2e_val else None, "unit": "GCUPS",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "how": "sw_search + sw_topk through the C-ABI with pinned host buffers, wall clock"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": per_step_kernels * args.steps + extra,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

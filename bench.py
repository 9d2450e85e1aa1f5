"""Benchmark: GCUPS of the B200 inter-task Smith-Waterman search
(BASELINE.json metric) on BASELINE.json configs[1] -- a query of 464 residues
against 1,000,000 synthetic sequences (~200 M residues), one B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 0|1|2|3|4]

A *step* is one pass of the whole hot path over the resident database
(SURVEY.md 8(a) rows a2-a6): query-profile build, the s16x2 pass kernel(s),
saturation flag compaction + exact s32 re-scoring, and the sorting stage
(device top-10).  Pre-processing (sw_db_load, row a1) is done once before the
timed region, as in the paper.  GCUPS = |Q||D| /
(t 1e9) (Eq. 4).

Multi-GPU: one process per GPU.  `--gpus N` without a
torchrun environment re-launches itself under torch.distributed.run with N
ranks.  Each rank generates and loads only its residue-balanced shard of the
database; a step is every rank's search of its shard, the NCCL gather of the
padded score vectors and top-10 candidates to rank 0, and on rank 0 the
device scatter of all scores to original database order plus the merged
top-10 (parallel.ShardedSearch).  Time = max over ranks of the device time.
  --config 0/1 (default 1): weak scaling, database = configs[k] x N.
  --config 2/3/4: strong scaling, the configuration's fixed database split
                  over the N ranks (configs[2]: 6.5 M sequences; configs[3]:
                  its 20 queries as query pairs, all in one step).
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
# biased arithmetic (unsigned or signed halves) 4.5 per 16x2 pair of cells (VIMNMX3 + 3 VIADDMNMX + 1/2
# VIMNMX3; the diagonal add runs on the FMA pipe), relu form 5.5 DPX.
ALU_PER_CELL = {2: 2.25, 1: 2.25, 0: 2.75}
WEAK_CONFIGS = (0, 1)


def parse(argv=None):
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
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: start N ranks (one process per GPU) with
    torch.distributed.run on this node; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    return {"sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md nominal clocks)"


def ncu_pipes():
    """ALU-pipe thread instructions per cell of the pass kernel, measured by ncu
    on the bench launch (profiles/ncu_pipes.json), for the roofline with
    the kernel's measured I_pipe."""
    for name in ("ncu_pipes.json", "r01b_ncu_pipes.json"):
        p = os.path.join(ROOT, "profiles", name)
        try:
            with open(p) as f:
                return json.load(f).get("alu_thread_inst_per_cell")
        except Exception:
            continue
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


def host_topk(x: np.ndarray, k: int) -> np.ndarray:
    """Indices of the k largest entries, score descending, index ascending
    (a host check of the device sorting stage, O(n))."""
    n = x.size
    kk = min(k, n)
    if kk == 0:
        return np.zeros(0, np.int64)
    thr = np.partition(x, n - kk)[n - kk]
    gt = np.nonzero(x > thr)[0]
    eq = np.nonzero(x == thr)[0][:kk - gt.size]
    cand = np.concatenate([gt, eq])
    return cand[np.lexsort((cand, -x[cand].astype(np.int64)))]


class Work:
    """One rank's share of a configuration's workload (see the module doc)."""

    def __init__(self, cfg: int, scale: float, world: int, rank: int, whole: bool = False):
        from paper_1702_07195_b200.parallel import shard_arrays, shard_database
        self.cfg = cfg
        self.weak = cfg in WEAK_CONFIGS
        gscale = scale * (world if self.weak else 1)
        if whole:   # the whole (global) database on this process (reference arm)
            world, rank = 1, 0
        if cfg == 4:   # built from a shuffled list: generate it whole (200 k sequences), then shard
            w = si.make_config(4, scale=gscale)
            lens, self.queries = w.db.lengths(), w.queries
            self.matrix, self.gap_open, self.gap_extend = w.matrix, w.gap_open, w.gap_extend
            self.gidx = shard_database(lens, world)[rank] if world > 1 else np.arange(lens.size, dtype=np.int64)
            res, offs = (shard_arrays(w.db.residues, w.db.offsets, self.gidx) if world > 1
                         else (w.db.residues, w.db.offsets))
            self.db = si.Database(res, offs)
        else:
            lens = si.config_lengths(cfg, gscale)
            self.queries = si.config_queries(cfg)
            self.matrix, self.gap_open, self.gap_extend = si.BLOSUM62, si.GAP_OPEN, si.GAP_EXTEND
            self.gidx = shard_database(lens, world)[rank] if world > 1 else np.arange(lens.size, dtype=np.int64)
            self.db = si.config_db_subset(cfg, self.gidx, gscale)
        self.count_global = int(lens.size)
        self.residues_global = int(lens.sum())
        wn = int(round(gscale / scale)) if self.weak else 1
        self.name = f"cfg{cfg}" + (f" x{wn} (weak)" if wn > 1 else "")
        if scale != 1.0:
            self.name += f" scale {scale}"
        self.qres = int(sum(len(q) for q in self.queries))

    def cells_global(self) -> int:
        return self.qres * self.residues_global


def cpu_baseline(w: Work, target_s: float = 12.0):
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
    return {"value": round(cells / dt / 1e9, 3), "unit": "GCUPS", "cores": cores, "cpu_model": cpu_model(),
            "kind": "oracle",
            "sample": f"{nsamp} seeded-random sequences of the workload ({int(lens[idx].sum())} residues) "
                      f"vs the {len(q)}-residue query 0 of the workload, {dt:.1f} s"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    w = Work(args.config, args.scale, world, 0, whole=True)
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
    sample = f"{nsamp} sequences per step (seeded, ~{budget:.0f} s each) of {w.name}, query 0 ({len(q)})"
    line = {"metric": METRIC, "value": round(val, 3), "unit": "GCUPS", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * total / max(1, len(times)), 3), "higher_is_better": True,
            "scaling": "weak" if args.config in WEAK_CONFIGS else "strong", "vs_baseline": None, "dtype": "i64",
            "data": "synthetic",
            "config": {"workload": workload_text(w, [q]), "query_len": len(q), "db_sequences": w.count_global,
                       "db_residues": w.residues_global},
            "cpu_baseline": {"value": round(val, 3), "unit": "GCUPS", "cores": cores, "cpu_model": cpu_model(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(val, 3), "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_text(w, queries):
    """The `config.workload` string, the same in both arms (the reference arm
    scores query 0 of the configuration only)."""
    nq = len(queries)
    qres = sum(len(q) for q in queries)
    return (f"{w.name}: {nq} quer{'y' if nq == 1 else 'ies'} ({qres} residues) vs "
            f"{w.count_global} synthetic sequences ({w.residues_global} residues), BLOSUM62, gaps 10/2")


def run_ours(args):
    import torch
    import paper_1702_07195_b200 as sw
    from paper_1702_07195_b200 import build as swbuild
    from paper_1702_07195_b200.parallel import LibBackend, ShardedSearch

    world, rank, local = dist_env()
    assert torch.cuda.is_available(), "bench needs a CUDA device"
    if world > torch.cuda.device_count():
        raise SystemExit(f"bench: {world} ranks but only {torch.cuda.device_count()} CUDA devices")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1 or args.dist:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
        print(f"[bench] rank {rank}/{world}: NCCL process group up on cuda:{local} "
              f"({torch.cuda.get_device_name(local)}), NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}",
              file=sys.stderr, flush=True)
    if args.gpus != world and rank == 0:
        print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE {world}; running {world} ranks",
              file=sys.stderr, flush=True)
    if rank == 0:
        swbuild.build()
    if dist:
        dist.barrier()

    w = Work(args.config, args.scale, world, rank)
    count = w.db.count
    local_res = w.db.total_residues
    sw.sw_db_load(w.db.residues, w.db.offsets)
    nq = len(w.queries)

    stream = torch.cuda.Stream(device=dev)
    search = ShardedSearch(LibBackend(sw), w.gidx, w.count_global, nq, TOPK, dev, dist=dist, world=world,
                           rank=rank)

    def step():
        return search.step(w.queries, w.matrix, w.gap_open, w.gap_extend, stream)

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    st = sw.sw_last_stats()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = sw.sw_launch_count()
    e0.record(stream)
    for i in range(args.steps):
        step()
        # the pass-kernel events of the last <= 64 searches are kept by the
        # library: read them every 64 steps (no synchronisation per step)
        if (i + 1) % 64 == 0:
            kernel_ms += sw.sw_timing_history(64)
    e1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    if args.steps % 64:
        kernel_ms += sw.sw_timing_history(args.steps % 64)
    launches = sw.sw_launch_count() - l0
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        tl = torch.tensor([float(launches)], dtype=torch.float64, device=dev)
        dist.all_reduce(tl, op=dist.ReduceOp.SUM)
        launches = int(tl.item())
    ms_step = ms_total / args.steps
    gcups = w.cells_global() / (ms_step * 1e6)

    # parity spot check of the assembled result on rank 0 (outside the timed region)
    checked = None
    if rank == 0:
        full, ti, ts = search.result()
        full_h = full.cpu().numpy()
        ok = bool(np.all(full_h >= 0))
        for qi in range(nq):
            order = host_topk(full_h[qi], search.kk)
            ok &= bool(np.array_equal(ti[qi].cpu().numpy(), order)
                       and np.array_equal(ts[qi].cpu().numpy(), full_h[qi][order]))
        checked = ok
        assert ok, "assembled scores and merged top-k disagree"

    # ---- end to end through the public C-ABI with host buffers
    e2e_val = None
    h2d = w.qres + 576
    d2h = nq * w.count_global * 4 + nq * TOPK * 12
    if world == 1 and nq == 1 and dist is None:
        # sw_search (pinned host scores) + sw_topk, wall clock
        host_scores = torch.empty(count, dtype=torch.int32, pin_memory=True).numpy()
        qpin = torch.empty(len(w.queries[0]), dtype=torch.uint8, pin_memory=True).numpy()
        qpin[:] = w.queries[0]
        mpin = torch.empty((24, 24), dtype=torch.int8, pin_memory=True).numpy()
        mpin[:] = w.matrix
        for _ in range(2):
            sw.sw_search(qpin, mpin, w.gap_open, w.gap_extend, out=host_scores)
            sw.sw_topk(TOPK)
        t0 = time.perf_counter()
        ne = max(3, args.steps // 3)
        for _ in range(ne):
            sw.sw_search(qpin, mpin, w.gap_open, w.gap_extend, out=host_scores)
            sw.sw_topk(TOPK)
        dt = (time.perf_counter() - t0) / ne
        e2e_how = "sw_search + sw_topk through the C-ABI with pinned host buffers, wall clock"
    else:
        # the sharded step with the host query (copied inside sw_search_dev), then
        # rank 0 reads all assembled scores and the top-k into pinned host memory
        if rank == 0:
            h_full = torch.empty(nq * w.count_global, dtype=torch.int32, pin_memory=True)
            h_ti = torch.empty((nq, TOPK), dtype=torch.int64, pin_memory=True)
            h_ts = torch.empty((nq, TOPK), dtype=torch.int32, pin_memory=True)

        def e2e_step():
            step()
            if rank == 0:
                with torch.cuda.stream(stream):
                    h_full.copy_(search.full, non_blocking=True)
                    h_ti.copy_(search.top_i, non_blocking=True)
                    h_ts.copy_(search.top_s, non_blocking=True)
            stream.synchronize()

        e2e_step()
        ne = max(3, args.steps // 3)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            e2e_step()
        if dist:
            dist.barrier()
        dt = (time.perf_counter() - t0) / ne
        e2e_how = ("sharded step through the C-ABI (host query) + NCCL gather + device assembly, then the "
                   "assembled scores and top-k D2H to pinned host memory on rank 0; wall clock between barriers")
    if dist:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    e2e_val = w.cells_global() / (dt * 1e9)

    # ---- roofline of the dominant kernel (s16x2 pass kernel, ALU/DPX bound)
    peaks, peaks_src = measured_peaks()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    kms = float(np.mean(kernel_ms))
    achieved = w.qres * local_res / (kms * 1e6)          # GCUPS of the pass kernels, this rank
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
    # HBM as the non-binding limit (north_star): algorithmic bytes per launch
    # (one pass over the shard: 1 B per residue + 4 B per score)
    # and the ncu DRAM traffic of the same launch against the measured copy bandwidth
    alg_bytes = int(local_res + 4 * w.db.count)
    hbm_peak = float(peaks.get("hbm_gbs", 0.0)) or None
    # the committed capture is of the default workload on one GPU
    tr = roof["traffic"] if (args.config == CONFIG_INDEX and world == 1 and args.scale == 1.0) else None
    roof["hbm"] = {"algorithmic_bytes": alg_bytes,
                   "algorithmic_GBps": round(alg_bytes / (kms * 1e6), 1),
                   "traffic_GBps": round(tr / (kms * 1e6), 1) if tr else None,
                   "peak_GBps": hbm_peak,
                   "frac": round(tr / (kms * 1e6) / hbm_peak, 4) if (tr and hbm_peak) else None,
                   "traffic_over_algorithmic": round(tr / alg_bytes, 2) if tr else None,
                   "traffic_is": "ncu dram bytes of the default workload's pass-kernel launch (profiles/ncu_summary.json)"}

    clk_all = None
    if dist:
        clk_all = [None] * world if rank == 0 else None
        dist.gather_object(clk, clk_all, dst=0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)

    if rank == 0:
        qlens = [len(q) for q in w.queries]
        line = {
            "metric": METRIC, "value": round(gcups, 1), "unit": "GCUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak" if w.weak else "strong", "vs_baseline": None,
            "dtype": "i16", "data": "synthetic",
            "config": {"workload": workload_text(w, w.queries),
                       "query_len": qlens[0] if nq == 1 else qlens, "db_sequences": w.count_global,
                       "db_residues": w.residues_global, "per_gpu_db_residues": local_res, "topk": TOPK,
                       "tile_G_R": [st["G"], st["R"]], "passes": st["passes"],
                       "flagged_rescored": st["flagged"],
                       "l2": "inputs larger than L2 (stream image %.0f MB > 126 MB)" % (st["pair_columns"] * 4 / 1e6),
                       "parallelism": f"dp{world} (database shards, one process per GPU)",
                       "ranks": world, "assembled_all_scores_on_rank0": True,
                       "assembly_check": checked},
            "e2e": {"value": round(e2e_val, 1) if e2e_val else None, "unit": "GCUPS",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "how": e2e_how},
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
        }
        if clk_all:
            line["clocks_per_rank"] = clk_all
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

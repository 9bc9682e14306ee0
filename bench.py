#!/usr/bin/env python3
"""Benchmark: split-FFT block-Toeplitz MVM/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c3|c3full|c2|c4|c1] [--no-e2e] [--no-cpu-baseline]
                    [--no-embed-baseline]

Default workload (N=1): BASELINE.json configs[3] — d=3, 512^3 grid, 3x3 dyadic
Green kernel (configs[1] definition), complex64, mirror-compressed spectra,
x i.i.d. CN(0,1) from the reference's RNG (seed 4); operators and inputs come
from paper_2406_17981_b200/workloads.py, the same ones the full-size parity
tests check against the reference (tests/test_fullsize_gpu.py). A "step" is
one MVM y = T x through the library's device API (ts_operator_apply_device).
At N>1 each rank owns 1/N of the 2^d branches (ts_split_options.part/nparts)
and ts_operator_apply_device_comm sums the projected partials with an NCCL
reduce inside the library, in the step. `--gpus N` outside torchrun launches
the N ranks itself.

Under torchrun (N>1) every rank runs; rank 0 prints ONE JSON line. The
reference arm (--impl reference) times the reference's own CPU code
(oracle/_ref, the unmodified reference compiled with an FFTW-API shim) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Toeplitz MVM/s at 512³ 3×3 c64, 1/2/4/8 B200; % of HBM roofline"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def b_alg(levels, m, m_unique, es, compressed):
    """Per-MVM algorithmic bytes: (4*2^d - 6) c s S_e + K."""
    d = len(levels)
    s = math.prod(levels)
    vec = (4 * 2 ** d - 6) * m * s * es
    if compressed:
        k = m_unique * math.prod(n + 1 for n in levels) * es
    else:
        k = m_unique * 2 ** d * s * es
    return vec + k, vec, k


def free_port():
    import socket

    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def self_launch(args):
    """--gpus N > 1 outside torchrun: launch N ranks (one per GPU) the way the
    driver does, and pass their output through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.run(cmd).returncode)


def family_profile(op, x, y, stream, steps):
    """Per-launch device times (CUDA events on the launching stream) over the
    same K MVMs, grouped by kernel family."""
    recs = []
    for _ in range(steps):
        recs += op.profile_device(x, y, stream)
    fam = {}
    for r in recs:
        key = {1: "fwd_split", 2: "leaf_pair", 3: "inv_merge"}.get(r["kind"], "other")
        f = fam.setdefault(key, {"ms": 0.0, "bytes": 0, "n": 0})
        f["ms"] += r["ms"]
        f["bytes"] += r["alg_bytes"]
        f["n"] += 1
    return fam


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2406_17981_b200 as T
    from paper_2406_17981_b200 import partition
    from paper_2406_17981_b200 import workloads as W

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    name = args.config
    levels, kind, prec, storage, _, _, cidx = W.CONFIGS[name]
    d = len(levels)
    s = math.prod(levels)
    partition.check_world(world, d)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- setup (not timed): operator with spectra precomputed on the device
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(dev)[0]
    mem0 = T.memory_stats(local)
    T.reset_memory_peak(local)
    t0 = time.time()
    if world > 1:
        pop = partition.PartitionedOperator(
            T, lambda r, w, dv: W.make_operator(T, name, part=r, nparts=w, device=dv),
            rank, world, local, d)
        op = pop.op
    else:
        pop = None
        op = W.make_operator(T, name, device=local)
    setup_s = time.time() - t0
    setup_peak = T.memory_stats(local)["peak_bytes"] - mem0["live_bytes"]
    info = op.info()
    m = info["m"]
    cdt = torch.complex64 if info["precision"] == T.C64 else torch.complex128
    xh = W.input_vector(T, name)  # reference RNG, complex128 host
    x = torch.from_numpy(xh).to(cdt).to(dev)  # rounded on the host: no complex128 device copy
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    def step():
        if pop is not None:
            pop.apply(x, y, stream)  # subtree + NCCL reduce of the partials (in the library)
        else:
            op.apply_device(x, y, stream)

    # ---- timed region: K MVMs on device-resident x, y
    T.reset_memory_peak(local)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ms_per_step = ms / args.steps
    value = args.steps / (ms / 1e3)  # MVM/s of the whole job

    # ---- device memory of the MVM, as the library meters it (spectra,
    # tables, the schedule's child buffers) plus the caller's x and y
    mem = T.memory_stats(local)
    info = op.info()
    peak_mvm = int(mem["peak_bytes"] + x.numel() * x.element_size() * 2)
    used_delta = int(free0 - torch.cuda.mem_get_info(dev)[0])

    # ---- per-launch profile for the roofline: the same K MVMs again with a
    # CUDA event pair around every launch (kept out of the timed loop)
    fam = family_profile(op, x, y, stream, args.steps)
    bw_peak, peak_src = peaks()
    dom = max(fam.items(), key=lambda kv: kv[1]["ms"])
    dom_bytes = dom[1]["bytes"] / dom[1]["n"]
    dom_ms = dom[1]["ms"] / dom[1]["n"]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    traffic = limiter = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            ent = json.load(f).get(name, {}).get(dom[0])
        if ent:
            traffic = ent.get("dram_bytes_per_launch")
            limiter = ent.get("limiter")
    es = info["elem_bytes"]
    compressed = info["storage"] == T.STORAGE_COMPRESSED
    balg, bvec, bk = b_alg(levels, m, info["n_unique"], es, compressed)

    # ---- end to end through the public API
    e2e = None
    if not args.no_e2e:
        if world == 1:
            e2e = e2e_abi(op, xh, args)
            e2e["device_api_pipelined"] = e2e_pipelined(op, x, y, xh, cdt, stream, args)
        else:
            e2e = e2e_comm(pop, x, y, xh, cdt, stream, args, rank, world, dev)

    # ---- the full-embedding cuFFT baseline (same run, same x), N=1
    emb = None
    if world == 1 and kind == "dyadic" and not args.no_embed_baseline:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import embed_baseline

        op.apply_device(x, y, stream)
        torch.cuda.synchronize()
        op.close()  # free the split operator's spectra and workspace first
        del op
        torch.cuda.empty_cache()
        try:
            emb = embed_baseline.run(levels, x, y, steps=max(2, min(args.steps, 5)), warmup=1)
            emb["peak_device_bytes_vs_split"] = emb["peak_device_bytes"] / peak_mvm
        except Exception as e:  # e.g. out of memory on a smaller GPU
            emb = {"unavailable": f"{type(e).__name__}: {e}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = reference_sample(args, name)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "MVM/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "c64" if info["precision"] == T.C64 else "c128",
            "data": "synthetic (reference SplitMix64/Box-Muller x, analytic dyadic kernel)"
                    if kind == "dyadic" else "synthetic (reference SplitMix64/Box-Muller lags and x)",
            "config": {
                "workload": f"BASELINE.json configs[{cidx}]: d={d} {'x'.join(map(str, levels))} "
                            f"{'3x3 dyadic' if kind == 'dyadic' else 'scalar'} {prec}, "
                            f"{'mirror-compressed' if compressed else 'full'} spectra",
                "levels": levels, "components": m, "unique_components": info["n_unique"],
                "storage": "compressed" if compressed else "full",
                "parallelism": f"branch partition over {world} GPUs, NCCL broadcast/reduce inside "
                               "libtoesplit (ts_operator_apply_device_comm)" if world > 1
                else "1 GPU, whole tree",
                "l2": "inputs (%.2f GB per vector) larger than the 126 MB L2; no flush needed"
                      % (m * s * es / 1e9) if m * s * es > 126e6 else
                      "working set partly L2-resident (vectors %.1f MB); no flush" % (m * s * es / 1e6),
                "B_alg_bytes_per_mvm": balg,
            },
            "roofline": {
                "bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": bw_peak,
                "unit": "GB/s", "frac": achieved / bw_peak, "traffic": traffic,
                "alg_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                "peak_source": peak_src, "limiter": limiter,
                "profiled_mvms": args.steps,
                "kernel_ms_per_mvm": sum(v["ms"] for v in fam.values()) / args.steps,
            },
            "step_roofline": {
                "B_alg_bytes": balg, "achieved_GBps": balg / (ms_per_step / 1e3) / 1e9 / world,
                "frac": balg / (ms_per_step / 1e3) / 1e9 / world / bw_peak,
                "per_gpu": world > 1,
            },
            "kernel_families": {k: {"launches": v["n"] // args.steps, "ms": v["ms"] / args.steps,
                                    "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9}
                                for k, v in fam.items()},  # per MVM (rank 0's share at N > 1)
            "gpu_launches": int(info["launches"]) * args.steps,
            "e2e": e2e,
            "embed_baseline": emb,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "peak_device_bytes": peak_mvm,
            "memory": {
                "peak_device_bytes": peak_mvm,
                "how": "libtoesplit device meter (ts_device_memory_stats peak over warm-up + timed "
                       "MVMs: spectra + tables + cached child buffers) + caller x and y",
                "library_peak_bytes": int(mem["peak_bytes"]),
                "spectra_bytes": int(info["spectra_bytes"]),
                "table_bytes": int(info["table_bytes"]),
                "workspace_bytes": int(info["cached_bytes"]),
                "x_y_bytes": int(2 * x.numel() * x.element_size()),
                "cuda_mem_get_info_delta_bytes": used_delta,
                "setup_peak_bytes": int(setup_peak),
                "per_gpu": world > 1,
            },
            "setup_s": setup_s,
        }
        print(json.dumps(line))
    if pop is not None:
        pop.close()
    if world > 1:
        dist.destroy_process_group()


def e2e_abi(op, xh, args):
    """The reference-facing call: ts_operator_apply on host complex128
    interleaved buffers (ref proj/include/toesplit.h:131-132), H2D / D2H and
    the precision conversion inside the call; the caller reuses its y."""
    import numpy as np

    ya = np.empty_like(xh)
    t = time.perf_counter()
    op.apply(xh, out=ya)  # first call: pinned staging pool, y pages touched
    first = time.perf_counter() - t
    ts = []
    for _ in range(max(2, min(args.steps, 5))):
        t = time.perf_counter()
        _, mt = op.apply(xh, out=ya, metrics=True)
        ts.append(time.perf_counter() - t)
    med = statistics.median(ts)
    return {"value": 1.0 / med, "unit": "MVM/s", "h2d_bytes_per_step": int(xh.nbytes),
            "d2h_bytes_per_step": int(ya.nbytes), "steps": len(ts), "seconds_per_call": ts,
            "first_call_s": first, "apply_ns_device": int(mt["apply_ns"]),
            "api": "ts_operator_apply (the reference ABI call): pageable host complex128 x in, "
                   "y out; staging, c128<->c64 rounding, H2D, MVM, D2H inside the call; "
                   "host wall clock per call, median"}


def e2e_pipelined(op, x, y, xh, cdt, stream, args):
    """Pinned host x -> device -> ts_operator_apply_device -> pinned host y
    every step, copies of neighbouring steps on two copy streams."""
    import torch

    dev = x.device
    xp = torch.from_numpy(xh).to(cdt).pin_memory()
    yp = torch.empty_like(xp).pin_memory()
    xs_ = [x, torch.empty_like(x)]
    ys_ = [y, torch.empty_like(y)]
    sh, sd = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    kp = max(3, args.steps)
    in_ev = [torch.cuda.Event() for _ in range(2)]
    used_ev = [torch.cuda.Event() for _ in range(2)]
    out_ev = [torch.cuda.Event() for _ in range(2)]
    done_ev = [torch.cuda.Event() for _ in range(2)]
    for e in used_ev + done_ev:
        e.record(stream)
    torch.cuda.synchronize()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(sh)
    for i in range(kp):
        b = i % 2
        sh.wait_event(used_ev[b])
        with torch.cuda.stream(sh):
            xs_[b].copy_(xp, non_blocking=True)
        in_ev[b].record(sh)
        stream.wait_event(in_ev[b])
        stream.wait_event(done_ev[b])
        op.apply_device(xs_[b], ys_[b], stream)
        used_ev[b].record(stream)
        out_ev[b].record(stream)
        sd.wait_event(out_ev[b])
        with torch.cuda.stream(sd):
            yp.copy_(ys_[b], non_blocking=True)
        done_ev[b].record(sd)
    p1.record(sd)
    torch.cuda.synchronize()
    val = kp / (p0.elapsed_time(p1) / 1e3)
    del xs_[1], ys_[1]
    return {"value": val, "unit": "MVM/s", "h2d_bytes_per_step": int(xp.numel() * xp.element_size()),
            "d2h_bytes_per_step": int(yp.numel() * yp.element_size()), "steps": kp,
            "api": "pinned host complex64 x -> ts_operator_apply_device -> pinned host y; copies of "
                   "neighbouring steps overlap on two copy streams (CUDA events)"}


def e2e_comm(pop, x, y, xh, cdt, stream, args, rank, world, dev):
    """N > 1: pinned host x -> rank 0 -> NCCL broadcast + subtrees + reduce
    (ts_operator_apply_device_comm) -> rank 0 -> pinned host y, every step."""
    import torch
    import torch.distributed as dist

    xp = torch.from_numpy(xh).to(cdt).pin_memory() if rank == 0 else None
    yp = torch.empty_like(xp).pin_memory() if rank == 0 else None

    def one():
        if rank == 0:
            x.copy_(xp, non_blocking=True)
        pop.apply(x, y, stream, bcast_x=True)
        if rank == 0:
            yp.copy_(y, non_blocking=True)

    one()
    torch.cuda.synchronize()
    dist.barrier()
    k = max(2, min(args.steps, 5))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    nb = x.numel() * x.element_size()
    return {"value": k / (float(t.item()) / 1e3), "unit": "MVM/s", "h2d_bytes_per_step": int(nb),
            "d2h_bytes_per_step": int(nb), "steps": k,
            "api": "pinned host x -> rank 0 -> ts_operator_apply_device_comm (NCCL broadcast, "
                   "subtrees, reduce) -> rank 0 -> pinned host y; serial, CUDA events, max over ranks"}


SAMPLE_N = {"c0": 16, "c1": 64, "c1m": 64, "c1_128": 64, "c2": 128, "c3": 128, "c3full": 128, "c4": 32}
CALIBRATION = os.path.join(ROOT, "profiles", "r02_reference_fullsize.json")


class RefSampler:
    """The UNMODIFIED reference (oracle/_ref) on host cores, on a bounded sample
    of the workload (same config, levels shrunk to sample_n per axis), built
    once; one() runs one sample MVM. Times are extrapolated to the full size
    with the reference's own C_split cost model (ts_predict) and, where a
    full-size run of the reference was measured on a box of this kind
    (profiles/r02_reference_fullsize.json), corrected by the model's measured
    error at that size."""

    def __init__(self, name, sample_n):
        import oracle
        from paper_2406_17981_b200 import workloads as W

        levels, kind, _, _, lag_seed, seed, _ = W.CONFIGS[name]
        self.name, self.levels, self.kind, self.n = name, levels, kind, sample_n
        d = len(levels)
        slv = [sample_n] * d
        self.ncores = os.cpu_count() or 1
        self.R = R = oracle.RefLib()
        O = oracle.Oracle()
        s = math.prod(slv)
        self.ops = []
        if kind == "dyadic":
            x = R.random_vector([3] + slv, seed, 0.5)
            self.xs = [x[i * s:(i + 1) * s] for i in range(3)]
            for i in range(3):
                for j in range(i, 3):
                    lags = O.dyadic_lags(slv, i, j)
                    g = R.generator(slv, lags, oracle.SYM_SYMMETRIC if i == j else oracle.SYM_GENERAL)
                    self.ops.append((i, j, R.split(g)))
                    R.destroy_gen(g)
        else:
            lags = O.random_lags(slv, lag_seed, 0.5, oracle.SYM_GENERAL)
            if kind == "scaled":
                lags = W.scale_lags_by_offset(lags, slv)
            g = R.generator(slv, lags, oracle.SYM_GENERAL)
            self.xs = R.random_vector(slv, seed, 0.5)
            self.ops.append((0, 0, R.split(g)))
            R.destroy_gen(g)
        self.s = s
        c_full = O.predict(d, float(levels[0]))["c_split"]
        c_samp = O.predict(d, float(sample_n))["c_split"]
        self.scale = c_full / c_samp
        self.calib = None
        if sample_n < levels[0] and os.path.exists(CALIBRATION):
            with open(CALIBRATION) as f:
                ent = json.load(f).get(name)
            if ent and ent.get("sample_n") == sample_n and ent.get("host_cores") == self.ncores:
                self.calib = ent

    def one(self, parallel=None, ops=None):
        import numpy as np

        R = self.R
        nc = self.ncores if parallel is None else parallel
        if ops is None:
            ops = self.ops
        t0 = time.perf_counter()
        if self.kind == "dyadic":
            ys = [np.zeros(self.s, np.complex128) for _ in range(3)]
            for i, j, op in ops:
                ys[i] += R.apply(op, self.xs[j], parallel=nc)
                if i != j:
                    ys[j] += R.apply(op, self.xs[i], parallel=nc)
        else:
            R.apply(ops[0][2], self.xs, parallel=nc)
        return time.perf_counter() - t0

    def full_seconds(self, t_sample):
        """Estimated seconds per full-size MVM from a sample time."""
        k = self.calib["model_correction"] if self.calib else 1.0
        return t_sample * self.scale * k

    def extras(self):
        """SURVEY.md §8(d) companions at the sample size: the same MVM with the
        LAZY policy (1 core) and with the reference's embedding engine (its
        CPU full-embedding path), each extrapolated with its own cost model."""
        import oracle

        out = {}
        t_lazy = self.one(parallel=0)
        out["lazy_1core"] = {"value": 1.0 / (t_lazy * self.scale), "sample_seconds": t_lazy}
        O = oracle.Oracle()
        d = len(self.levels)
        slv = [self.n] * d
        emb = []
        try:
            if self.kind == "dyadic":
                for i in range(3):
                    for j in range(i, 3):
                        g = self.R.generator(slv, O.dyadic_lags(slv, i, j), oracle.SYM_GENERAL)
                        emb.append((i, j, self.R.embed(g)))
                        self.R.destroy_gen(g)
            else:
                g = self.R.generator(slv, seed=5, symmetry=0, variance=0.5)
                emb.append((0, 0, self.R.embed(g)))
                self.R.destroy_gen(g)
            t_emb = self.one(ops=emb)
            ce = O.predict(d, float(self.levels[0]))["c_embed"] / O.predict(d, float(self.n))["c_embed"]
            out["embed_engine"] = {"value": 1.0 / (t_emb * ce), "sample_seconds": t_emb,
                                   "note": "reference CPU full-embedding engine, same composition, "
                                           f"extrapolated x{ce:.1f} by its C_embed model"}
        finally:
            for _, _, op in emb:
                self.R.destroy_op(op)
        return out

    def close(self):
        for _, _, op in self.ops:
            self.R.destroy_op(op)
        self.ops = []

    def describe(self, t, reps):
        d = len(self.levels)
        what = ("3x3 dyadic (9 scalar reference applies, G_ii symmetric, G_ij general)"
                if self.kind == "dyadic" else "scalar")
        full = self.full_seconds(t)
        out = {
            "value": 1.0 / full, "unit": "MVM/s", "cores": self.ncores, "kind": "reference",
            "sample": f"{what} MVM at {self.n}^{d}, c128 (the reference's only precision), "
                      f"TS_POLICY_PARALLEL task_budget={self.ncores}; median {t:.3f} s over {reps} rep(s)"
                      + (f", extrapolated x{self.scale:.1f} to {self.levels[0]}^{d} by the reference's "
                         "C_split model" if self.scale != 1.0 else " (full size)")
                      + (f" and corrected x{self.calib['model_correction']:.3f} by the model's error "
                         "against a measured full-size run" if self.calib else ""),
            "sample_seconds": t,
            "full_size_seconds_estimate": full,
            "fft": "reference engine + substitute FFT (FFTW-API shim, FFTW3 absent)",
        }
        if self.calib:
            out["calibration"] = self.calib
        return out


def ref_sample_n(name):
    return int(os.environ.get("TS_REF_SAMPLE_N", SAMPLE_N.get(name, 128)))


def reference_sample(args, name, budget_s=12.0):
    """cpu_baseline: repeat the sample MVM for about budget_s seconds of CPU work."""
    try:
        smp = RefSampler(name, ref_sample_n(name))
    except Exception as e:  # reference build absent
        return {"unavailable": f"oracle/_ref not built: {e}"}
    try:
        ts = [smp.one()]
        reps = max(1, min(20, int(budget_s / max(ts[0], 1e-3))))
        ts += [smp.one() for _ in range(reps - 1)]
        out = smp.describe(statistics.median(ts), len(ts))
        try:
            out.update(smp.extras())
        except Exception as e:  # companions are informational
            out["extras_error"] = str(e)
        return out
    finally:
        smp.close()


def run_reference(args):
    from paper_2406_17981_b200 import workloads as W

    world, rank, _ = dist_env()
    if rank != 0:
        return
    name = args.config
    levels, kind, prec, _, _, _, cidx = W.CONFIGS[name]
    t0 = time.perf_counter()
    try:
        smp = RefSampler(name, ref_sample_n(name))
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    per = []
    for i in range(args.warmup + args.steps):
        t = smp.one()
        if i >= args.warmup:
            per.append(smp.full_seconds(t))
    smp.close()
    base = smp.describe(statistics.median(per) / (smp.full_seconds(1.0)), len(per))
    t_step = statistics.mean(per)
    value = 1.0 / t_step
    base["value"] = value
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "MVM/s",
        "n_gpus": args.gpus, "host_cores": os.cpu_count(), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (reference SplitMix64/Box-Muller x, analytic dyadic kernel)",
        "config": {"workload": f"BASELINE.json configs[{cidx}] on host cores (sampled)",
                   "levels": levels},
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "MVM/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line))


def main():
    from paper_2406_17981_b200 import workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(W.CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-embed-baseline", action="store_true",
                    help="skip the full-embedding cuFFT MVM (dyadic configs; ~110 GB at 512^3)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("note: the timing rules ask for >= 3 warm-up steps", file=sys.stderr)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        self_launch(args)  # the reference arm is rank 0's host cores only: nothing to launch
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Benchmark: split-FFT block-Toeplitz MVM/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c3|c3full|c2|c4|c1] [--no-e2e] [--no-cpu-baseline] [--embed-baseline]

Default workload (N=1): BASELINE.json configs[3] — d=3, 512^3 grid, 3x3 dyadic
Green kernel (configs[1] definition), complex64, mirror-compressed spectra,
x i.i.d. CN(0,1) from the reference's RNG (seed 4). A "step" is one MVM
y = T x through the library's device API (ts_operator_apply_device); at N>1
each rank owns 1/N of the 2^d branches (ts_split_options.part/nparts) and the
projected partials are summed with an NCCL reduce inside the step.

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

CONFIGS = {
    # name: (levels, kind, precision, storage, x seed, BASELINE configs index)
    "c3": ([512, 512, 512], "dyadic", "c64", "auto", 4, 3),
    "c3full": ([512, 512, 512], "dyadic", "c64", "full", 4, 3),  # full 6-unique spectra
    "c2": ([256, 256, 256], "dyadic", "c64", "auto", 3, 2),
    "c1": ([64, 64, 64], "dyadic", "c64", "full", 2, 1),
    "c4": ([64, 64, 64, 64], "scalar", "c64", "full", 6, 4),
}
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
            self._stop.wait(0.2)

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


def make_operator(T, cfg, part, nparts, device):
    levels, kind, prec, storage, _, _ = cfg
    st = {"auto": T.STORAGE_AUTO, "full": T.STORAGE_FULL, "compressed": T.STORAGE_COMPRESSED}[storage]
    pr = T.C64 if prec == "c64" else T.C128
    if kind == "dyadic":
        bg = T.BlockGenerator.dyadic(levels)
    else:
        bg = None
    if bg is None:
        # configs[4]: non-symmetric CN(0,1) lags scaled by 1/(1+|m|_2), seed 5
        import numpy as np
        g = T.Generator.random(levels, 5, 0.5, T.SYM_GENERAL)
        lags = g.lags()
        grids = np.meshgrid(*[np.arange(-(n - 1), n) for n in levels], indexing="ij")
        r = np.sqrt(sum(gr.astype(np.float64) ** 2 for gr in grids)).reshape(-1)
        lags = lags / (1.0 + r)
        bg = T.BlockGenerator.create(levels, 1, [0], [lags], [[0] * len(levels)])
        del g
    return T.Operator.split_ex(bg, precision=pr, storage=st, device=device, part=part,
                               nparts=nparts)


def gen_input(T, cfg):
    """x i.i.d. CN(0,1) (variance 0.5 per part) from the reference RNG, SoA."""
    import numpy as np
    levels, kind, _, _, seed, _ = cfg
    comp = 3 if kind == "dyadic" else 1
    lv = ([comp] + list(levels)) if comp > 1 else list(levels)
    return T.random_vector(lv, seed, 0.5).astype(np.complex128, copy=False)


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2406_17981_b200 as T

    world, rank, local = dist_env()
    if world != args.gpus:
        if not (world == 1 and args.gpus == 1):
            print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    levels, kind, prec, storage, seed, cidx = cfg
    d = len(levels)
    if world > 2 ** d:
        raise SystemExit(f"at most 2^d = {2 ** d} GPUs (one branch each)")

    t0 = time.time()
    op = make_operator(T, cfg, rank, world, local)
    setup_s = time.time() - t0
    info = op.info()
    m = info["m"]
    s = math.prod(levels)
    cdt = torch.complex64 if info["precision"] == T.C64 else torch.complex128
    xh = gen_input(T, cfg)
    x = torch.from_numpy(xh).to(dev).to(cdt)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    from paper_2406_17981_b200 import partition

    partition.check_world(world, d)

    def step():
        op.apply_device(x, y, stream)
        if world > 1:
            partition.reduce_partials(y, dst=0)  # NCCL over NVLink

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ms_per_step = ms / args.steps
    value = args.steps / (ms / 1e3)  # MVM/s (one MVM per step for the whole job)

    # per-launch profile for the roofline: the same K MVMs again, with a CUDA
    # event pair around every launch on the launching stream (kept out of the
    # timed loop above so that `value` carries no event overhead)
    recs = []
    for _ in range(args.steps):
        recs += op.profile_device(x, y, stream)
    fam = {}
    for r in recs:
        key = {1: "fwd_split", 2: "leaf_pair", 3: "inv_merge"}.get(r["kind"], "other")
        f = fam.setdefault(key, {"ms": 0.0, "bytes": 0, "n": 0})
        f["ms"] += r["ms"]
        f["bytes"] += r["alg_bytes"]
        f["n"] += 1
    bw_peak, peak_src = peaks()
    dom = max(fam.items(), key=lambda kv: kv[1]["ms"])
    dom_bytes = dom[1]["bytes"] / dom[1]["n"]
    dom_ms = dom[1]["ms"] / dom[1]["n"]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    traffic = None
    limiter = None  # what bounds the dominant kernel when HBM does not (ncu pipes)
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        ent = tj.get(args.config, {}).get(dom[0])
        if ent:
            traffic = ent.get("dram_bytes_per_launch")
            limiter = ent.get("limiter")
    es = info["elem_bytes"]
    compressed = info["storage"] == T.STORAGE_COMPRESSED
    balg, bvec, bk = b_alg(levels, m, info["n_unique"], es, compressed)

    # device memory of the MVM itself (operator + x, y + stream-ordered workspace),
    # before the e2e section adds its second x/y pair
    peak_mvm = torch.cuda.max_memory_allocated(dev)

    # end-to-end through the public API: pinned host x -> device -> MVM
    # (+ reduce) -> pinned host y, every step
    e2e = None
    if not args.no_e2e:
        xp = torch.from_numpy(xh).to(cdt).pin_memory()
        yp = torch.empty_like(xp).pin_memory()
        ke = max(1, min(args.steps, 3))

        def e2e_step():
            x.copy_(xp, non_blocking=True)
            step()
            if rank == 0:
                yp.copy_(y, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        serial = ke / (float(ems.item()) / 1e3)
        # pipelined across steps (how a serving loop would run it): H2D of step
        # i+1 and D2H of step i-1 on their own copy streams (separate copy
        # engines) while step i computes; two x and two y device buffers.
        # Every step still moves its whole x in and its whole y out.
        xs_ = [x, torch.empty_like(x)]
        ys_ = [y, torch.empty_like(y)]
        sh = torch.cuda.Stream(dev)
        sd = torch.cuda.Stream(dev)
        kp = max(3, args.steps)  # the same K steps as the device-resident number
        in_ev = [torch.cuda.Event() for _ in range(2)]
        used_ev = [torch.cuda.Event() for _ in range(2)]
        out_ev = [torch.cuda.Event() for _ in range(2)]
        done_ev = [torch.cuda.Event() for _ in range(2)]
        for e in used_ev + done_ev:
            e.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
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
            if world > 1:
                partition.reduce_partials(ys_[b], dst=0)
            used_ev[b].record(stream)
            out_ev[b].record(stream)
            sd.wait_event(out_ev[b])
            if rank == 0:
                with torch.cuda.stream(sd):
                    yp.copy_(ys_[b], non_blocking=True)
            done_ev[b].record(sd)
        p1.record(sd)
        torch.cuda.synchronize()
        pms = torch.tensor([p0.elapsed_time(p1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(pms, op=dist.ReduceOp.MAX)
        e2e = {"value": kp / (float(pms.item()) / 1e3), "unit": "MVM/s",
               "h2d_bytes_per_step": int(xp.numel() * xp.element_size()),
               "d2h_bytes_per_step": int(yp.numel() * yp.element_size()),
               "steps": kp, "serial_value": serial,
               "api": "pinned host x -> ts_operator_apply_device (+NCCL reduce) -> pinned host y; "
                      "copies of neighbouring steps overlap on two copy streams (serial_value: "
                      "one stream, no overlap)"}
        del xs_[1], ys_[1]
        # the reference-facing C-ABI call (ts_operator_apply, host complex128
        # interleaved doubles, H2D/D2H inside the call) at N=1
        if world == 1 and not args.no_abi_e2e:
            xa = xh
            t1 = time.perf_counter()
            ya = op.apply(xa)
            e2e["abi_ts_operator_apply_s"] = time.perf_counter() - t1
            e2e["abi_h2d_bytes"] = int(xa.nbytes)
            del ya
        del xp, yp

    emb = None
    if args.embed_baseline and kind == "dyadic" and world == 1:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import embed_baseline

        op.apply_device(x, y, stream)
        torch.cuda.synchronize()
        emb = embed_baseline.run(levels, x, y)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = reference_sample(args, cfg)

    peak_mem = peak_mvm
    peak_all = torch.cuda.max_memory_allocated(dev)
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
            "data": "synthetic (reference SplitMix64/Box-Muller x, analytic dyadic kernel)",
            "config": {
                "workload": f"BASELINE.json configs[{cidx}]: d={d} {'x'.join(map(str, levels))} "
                            f"{'3x3 dyadic' if kind == 'dyadic' else 'scalar'} {prec}, "
                            f"{'mirror-compressed' if compressed else 'full'} spectra",
                "levels": levels, "components": m, "unique_components": info["n_unique"],
                "storage": "compressed" if compressed else "full",
                "parallelism": f"branch partition over {world} GPU(s) + NCCL reduce" if world > 1
                else "1 GPU, whole tree",
                "l2": "inputs (%.2f GB per vector) larger than the 126 MB L2; no flush needed"
                      % (m * s * es / 1e9),
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
                                for k, v in fam.items()},  # per MVM
            "gpu_launches": int(info["launches"]) * args.steps,
            "e2e": e2e,
            "embed_baseline": emb,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "peak_device_bytes": int(peak_mem),
            "peak_device_bytes_incl_e2e_buffers": int(peak_all),
            "spectra_bytes": int(info["spectra_bytes"]),
            "setup_s": setup_s,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


class RefSampler:
    """The UNMODIFIED reference (oracle/_ref) on host cores, on a bounded sample
    of the workload (same config, levels shrunk to sample_n per axis), built
    once; one() runs one sample MVM. Times are extrapolated to the full size
    with the reference's own C_split cost model (ts_predict)."""

    def __init__(self, cfg, sample_n):
        import numpy as np

        import oracle

        levels, kind, _, _, seed, _ = cfg
        self.levels, self.kind, self.n = levels, kind, sample_n
        d = len(levels)
        slv = [sample_n] * d
        self.ncores = os.cpu_count() or 1
        self.R = R = oracle.RefLib()
        O = oracle.Oracle()
        s = math.prod(slv)
        self.ops = []
        if kind == "dyadic":
            x = O.random_vector([3] + slv, seed, 0.5)
            self.xs = [x[i * s:(i + 1) * s] for i in range(3)]
            for i in range(3):
                for j in range(i, 3):
                    lags = O.dyadic_lags(slv, i, j)
                    g = R.generator(slv, lags, oracle.SYM_SYMMETRIC if i == j else oracle.SYM_GENERAL)
                    self.ops.append((i, j, R.split(g)))
                    R.destroy_gen(g)
        else:
            g = R.generator(slv, seed=5, symmetry=0, variance=0.5)
            self.xs = R.random_vector(slv, seed, 0.5)
            self.ops.append((0, 0, R.split(g)))
            R.destroy_gen(g)
        self.s = s
        c_full = O.predict(d, float(levels[0]))["c_split"]
        c_samp = O.predict(d, float(sample_n))["c_split"]
        self.scale = c_full / c_samp

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
        return {
            "value": 1.0 / (t * self.scale), "unit": "MVM/s", "cores": self.ncores, "kind": "reference",
            "sample": f"{what} MVM at {self.n}^{d}, c128 (the reference's only precision), "
                      f"TS_POLICY_PARALLEL task_budget={self.ncores}; median {t:.3f} s over {reps} rep(s), "
                      f"extrapolated x{self.scale:.1f} to {self.levels[0]}^{d} by the reference's C_split model",
            "sample_seconds": t,
            "fft": "reference engine + substitute FFT (FFTW-API shim, FFTW3 absent)",
        }


def ref_sample_n():
    return int(os.environ.get("TS_REF_SAMPLE_N", "128"))


def reference_sample(args, cfg, budget_s=12.0):
    """cpu_baseline: repeat the sample MVM for about budget_s seconds of CPU work."""
    try:
        smp = RefSampler(cfg, ref_sample_n())
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
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    levels, kind, prec, _, _, cidx = cfg
    t0 = time.perf_counter()
    try:
        smp = RefSampler(cfg, ref_sample_n())
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    per = []
    for i in range(args.warmup + args.steps):
        t = smp.one()
        if i >= args.warmup:
            per.append(t * smp.scale)
    smp.close()
    base = smp.describe(statistics.median(per) / smp.scale, len(per))
    t_step = statistics.mean(per)
    value = 1.0 / t_step
    base["value"] = value
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "MVM/s",
        "n_gpus": args.gpus, "host_cores": os.cpu_count(), "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-abi-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--embed-baseline", action="store_true",
                    help="also time the full-embedding MVM with cuFFT (dyadic configs; ~120 GB)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("note: the timing rules ask for >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

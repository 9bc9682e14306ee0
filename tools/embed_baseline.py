"""Full circulant-embedding MVM on the GPU with cuFFT (torch.fft) — the method
the split-FFT paper improves on — as a comparison point for bench.py
(--embed-baseline) and an independent full-size cross-check of the split
engine's output. Not product code; the product path never calls this.

Dyadic 3x3 block kernel (BASELINE.json configs[1]): G_ij(m) =
(d_ij - r_i r_j / r^2) e^{ikr}/r + (d_ij - 3 r_i r_j / r^2) e^{ikr}/(k^2 r^3),
G(0) = self * I, evaluated on the 2n-periodic embedding (padding plane j = n
set to 0, the reference's default s0), transformed in complex128 once, kept in
complex64. One MVM: zero-pad x to (2n)^d, forward FFTs, 3x3 multiply, inverse
FFTs, crop — all complex64 cuFFT.
"""
import math
import time

import torch


def dyadic_spectra(levels, k=2 * math.pi / 10, self_term=1 + 0.1j, dev="cuda"):
    d = len(levels)
    assert d == 3
    n2 = [2 * n for n in levels]
    axes = []
    pads = []
    for n in levels:
        j = torch.arange(2 * n, device=dev, dtype=torch.float64)
        m = torch.where(j < n, j, j - 2 * n)
        axes.append(m)
        pads.append(j == n)
    spectra = {}
    for i in range(3):
        for jj in range(i, 3):
            out = torch.empty(n2, dtype=torch.complex128, device=dev)
            delta = 1.0 if i == jj else 0.0
            for a0 in range(n2[0]):  # slab by slab: bounded temporaries
                m0 = axes[0][a0]
                m1 = axes[1].view(-1, 1)
                m2 = axes[2].view(1, -1)
                r2 = m0 * m0 + m1 * m1 + m2 * m2
                comps = [m0.expand_as(r2), m1.expand_as(r2), m2.expand_as(r2)]
                rr = comps[i] * comps[jj] / torch.where(r2 == 0, torch.ones_like(r2), r2)
                r = torch.sqrt(r2)
                rs = torch.where(r2 == 0, torch.ones_like(r), r)
                amp = (delta - rr) / rs + (delta - 3.0 * rr) / (k * k * rs * rs * rs)
                v = torch.polar(amp, k * r)
                v = torch.where(r2 == 0, torch.full_like(v, delta * self_term), v)
                pad = pads[0][a0] | pads[1].view(-1, 1) | pads[2].view(1, -1)
                v = torch.where(pad, torch.zeros_like(v), v)
                out[a0] = v
            spectra[(i, jj)] = torch.fft.fftn(out).to(torch.complex64)
            del out
            torch.cuda.empty_cache()
    return spectra


def embed_apply(levels, spectra, xs):
    """xs: 3 complex64 tensors of shape levels -> 3 outputs (same shape)."""
    n0, n1, n2 = levels
    X = []
    for x in xs:
        p = torch.zeros((2 * n0, 2 * n1, 2 * n2), dtype=torch.complex64, device=x.device)
        p[:n0, :n1, :n2] = x
        X.append(torch.fft.fftn(p))
        del p
    ys = []
    for i in range(3):
        acc = None
        for j in range(3):
            t = spectra[(min(i, j), max(i, j))]
            term = t * X[j]
            acc = term if acc is None else acc.add_(term)
            del term
        y = torch.fft.ifftn(acc)
        del acc
        ys.append(y[:n0, :n1, :n2].contiguous())
        del y
    return ys


def run(levels, x_flat, y_ref_flat, steps=3, warmup=1):
    """Time the embedding MVM (device-resident x, CUDA events) and compare
    its output with the split engine's y. Returns a dict for the bench line.

    peak_device_bytes: the embedding's own high-water mark (torch caching
    allocator, which also serves cuFFT's plan workspace: spectra, padded
    vectors, products, outputs) plus its input x — comparable with the split
    engine's metered peak + x + y."""
    s = math.prod(levels)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    free0 = torch.cuda.mem_get_info()[0]
    t0 = time.time()
    spectra = dyadic_spectra(levels)
    setup = time.time() - t0
    xs = [x_flat[c * s:(c + 1) * s].view(*levels) for c in range(3)]
    for _ in range(warmup):
        ys = embed_apply(levels, spectra, xs)
        del ys
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()  # the MVM's peak (the setup transients are larger)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        ys = embed_apply(levels, spectra, xs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    peak_own = torch.cuda.max_memory_allocated() - base
    used = free0 - torch.cuda.mem_get_info()[0]
    y = torch.cat([v.reshape(-1) for v in ys])
    yr = y_ref_flat.to(torch.complex128)
    err = (torch.linalg.vector_norm(y.to(torch.complex128) - yr) / torch.linalg.vector_norm(yr)).item()
    del spectra, ys, y, yr
    torch.cuda.empty_cache()
    xbytes = x_flat.numel() * x_flat.element_size()
    return {"value": 1e3 / ms, "unit": "MVM/s", "ms_per_step": ms, "steps": steps,
            "impl": "full (2n)^3 circulant embedding, complex64 cuFFT via torch.fft (spectra "
                    "from complex128), 6 unique 3x3 spectra resident",
            "setup_s": setup, "rel_l2_vs_split_engine": err,
            "peak_device_bytes": int(peak_own + xbytes),
            "peak_how": "torch allocator high-water mark over the timed MVMs (spectra, padded "
                        "vectors, products, cuFFT workspace, outputs) + input x",
            "cuda_mem_get_info_delta_bytes": int(used)}

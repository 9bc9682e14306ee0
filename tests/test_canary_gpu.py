"""Out-of-bounds write check without compute-sanitizer (closed on the GPU pool): y (and the
multi-RHS y) sits inside one larger device buffer whose bytes before and after it hold a
pattern; after applies through every kernel family the pattern must be intact, x must be
unchanged (the passes run in place on child buffers, never on the caller's x), and the result
must equal the one computed into a plain buffer."""
import numpy as np
import pytest

import paper_2406_17981_b200 as T

pytestmark = pytest.mark.gpu

GUARD = 1 << 16  # complex elements on each side

CASES = [
    # (levels, block generator kind, precision): one per kernel family
    ([512, 512], "scalar", T.C64),        # TMA strided passes + 512-point leaf
    ([256, 256], "scalar", T.C64),        # 256-point passes
    ([64, 64, 64], "dyadic", T.C64),      # 3x3 leaf, compressed spectra
    ([8, 16, 512], "dyadic", T.C64),      # 512-point 3x3 leaf
    ([16, 8, 256], "dyadic", T.C64),
    ([128, 32, 64], "scalar", T.C128),    # complex128 fast passes
    ([12, 40, 36], "scalar", T.C128),     # mixed radix
    ([13, 64, 10], "scalar", T.C64),      # prime axis
    ([3, 4099], "scalar", T.C64),         # long prime axis (global-memory passes)
    ([2, 3, 8192], "scalar", T.C64),      # long power-of-two axis
    ([5, 4, 3, 6, 2], "scalar", T.C128),  # d = 5
    ([1, 7, 1], "scalar", T.C64),         # length-1 axes
]


@pytest.mark.parametrize("levels,kind,prec", CASES)
def test_no_write_outside_y(levels, kind, prec):
    import torch

    if kind == "dyadic":
        bg, m = T.BlockGenerator.dyadic(levels), 3
    else:
        bg, m = T.BlockGenerator.from_scalar(T.Generator.random(levels, 9, 1.0, T.SYM_SYMMETRIC)), 1
    op = T.Operator.split_ex(bg, precision=prec)
    dt = torch.complex64 if prec == T.C64 else torch.complex128
    n = m * int(np.prod(levels))
    gen = torch.Generator("cuda").manual_seed(1234)
    for nrhs in (1, 3):
        x = torch.randn(n * nrhs, dtype=dt, device="cuda", generator=gen)
        x0 = x.clone()
        plain = torch.empty_like(x)
        big = torch.empty(n * nrhs + 2 * GUARD, dtype=dt, device="cuda")
        pattern = torch.randn(2 * GUARD, dtype=dt, device="cuda", generator=gen)
        big[:GUARD] = pattern[:GUARD]
        big[GUARD + n * nrhs:] = pattern[GUARD:]
        y = big[GUARD:GUARD + n * nrhs]
        if nrhs == 1:
            op.apply_device(x, plain)
            op.apply_device(x, y)
        else:
            op.apply_batch_device(x, plain, nrhs)
            op.apply_batch_device(x, y, nrhs)
        torch.cuda.synchronize()
        assert torch.equal(big[:GUARD], pattern[:GUARD]), "write before y"
        assert torch.equal(big[GUARD + n * nrhs:], pattern[GUARD:]), "write after y"
        assert torch.equal(x, x0), "x modified"
        assert torch.equal(y, plain)
        assert bool(torch.isfinite(torch.view_as_real(y)).all())


def test_misaligned_device_pointers_are_rejected_not_faulted():
    # the fast passes use 16-byte vector accesses and bulk row copies: an x or y that is only
    # 8-byte aligned (a complex64 view at an odd element offset) is refused at the ABI
    # (TS_ERR_INVALID_ARGUMENT) instead of faulting in a kernel; aligned views work
    import torch

    levels = [8, 16, 512]
    op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=T.C64)
    n = 3 * int(np.prod(levels))
    x = torch.randn(n + 8, dtype=torch.complex64, device="cuda")
    y = torch.zeros(n + 8, dtype=torch.complex64, device="cuda")
    ref = torch.empty(n, dtype=torch.complex64, device="cuda")
    op.apply_device(x[2:2 + n], ref)
    for ox, oy in ((3, 0), (2, 1), (3, 5)):
        with pytest.raises(T.TsError) as e:
            op.apply_device(x[ox:ox + n], y[oy:oy + n])
        assert e.value.code == T.TS_ERR_INVALID_ARGUMENT
    op.apply_device(x[2:2 + n], y[4:4 + n])
    torch.cuda.synchronize()
    assert torch.equal(y[4:4 + n], ref)
    assert float(y[:4].abs().sum()) == 0 and float(y[4 + n:].abs().sum()) == 0

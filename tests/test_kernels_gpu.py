"""Kernel seams on the GPU vs the reference's outputs (golden fixtures) and
the oracle. Bit-exact comparisons throughout."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ring as oring
from tests.golden.gen import quant_cases
from tests.gpu_util import bits, need_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


@pytest.mark.parametrize("dt", ["float32", "float64"])
@pytest.mark.parametrize("opname", ["add", "max", "min"])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_accumulate_edges_match_reference(edges_npz, dt, opname, offset):
    from paper_2505_14065_b200 import accumulate

    a = edges_npz[f"{dt}__a"][offset:]
    b = edges_npz[f"{dt}__b"][offset:]
    want = edges_npz[f"{dt}__{opname}"][offset:]
    # offset views exercise the scalar head / misaligned paths
    big_a = to_dev(np.concatenate([np.zeros(offset, a.dtype), a]))
    big_b = to_dev(np.concatenate([np.zeros(offset, b.dtype), b]))
    da, db = big_a[offset:], big_b[offset:]
    accumulate({"add": "sum", "max": "max", "min": "min"}[opname], da, db)
    torch.cuda.synchronize()
    assert bits(da) == bits(want)


@pytest.mark.parametrize("dt", ["float32", "float64"])
@pytest.mark.parametrize("w", [3, 7])
def test_finalize_avg_matches_reference(edges_npz, dt, w):
    from paper_2505_14065_b200 import finalize_reduction

    a = to_dev(edges_npz[f"{dt}__a"])
    finalize_reduction(a, "avg", w)
    assert bits(a) == bits(edges_npz[f"{dt}__div{w}"])
    s = to_dev(edges_npz[f"{dt}__a"])
    finalize_reduction(s, "sum", w)
    assert bits(s) == bits(edges_npz[f"{dt}__a"])


def test_quantize_cases_match_reference(golden, quant_npz):
    from paper_2505_14065_b200 import dequantize_into, quantize_chunk

    meta = {m["name"]: m for m in golden["quant"]}
    for name, values in quant_cases():
        m = meta[name]
        x = to_dev(values)
        codes = torch.empty(max(values.size, 1), dtype=torch.uint8, device="cuda")
        if "error" in m:
            with pytest.raises(ValueError):
                quantize_chunk(x, codes)
            continue
        mn, sc = quantize_chunk(x, codes)
        assert (mn, sc) == (m["min"], m["scale"]), name
        assert bits(codes[: values.size]) == bits(quant_npz[f"{name}__q"]), name
        back = torch.empty_like(x)
        dequantize_into(codes, mn, sc, back)
        assert bits(back) == bits(quant_npz[f"{name}__d"]), name


@pytest.mark.parametrize("offset", [1, 2, 3, 5])
def test_quantize_misaligned_views(offset):
    from paper_2505_14065_b200 import quantize_chunk

    rng = np.random.default_rng(offset)
    v = rng.normal(0, 3, 100_003).astype(np.float32)
    want = np.empty(v.size, np.uint8)
    wmn, wsc = oring.quantize_chunk(v, want)
    x = to_dev(np.concatenate([np.zeros(offset, np.float32), v]))[offset:]
    codes = torch.zeros(v.size + 7, dtype=torch.uint8, device="cuda")[offset % 4 + 1 :][: v.size]
    mn, sc = quantize_chunk(x, codes)
    assert (mn, sc) == (wmn, wsc)
    assert bits(codes) == bits(want)


@pytest.mark.parametrize("opname", ["sum", "max", "min"])
def test_dequant_accumulate_with_range(opname):
    from paper_2505_14065_b200.collective import QuantScratch, dequant_accumulate, quantize_chunk_async

    rng = np.random.default_rng(11)
    n = 1_000_001
    x = rng.normal(0, 1, n).astype(np.float32)
    acc = rng.normal(0, 1, n).astype(np.float32)
    codes = np.empty(n, np.uint8)
    mn, sc = oring.quantize_chunk(x, codes)
    part = np.empty(n, np.float32)
    oring.dequantize_into(codes, mn, sc, part)
    want = acc.copy()
    oring.accumulate(oring.ReduceOp[opname.upper()], want, part)

    dx = to_dev(x)
    dcodes = torch.empty(n, dtype=torch.uint8, device="cuda")
    scratch = QuantScratch("cuda")
    quantize_chunk_async(dx, dcodes, scratch)
    dacc = to_dev(acc)
    nxt = torch.zeros(4, dtype=torch.int32, device="cuda")
    dequant_accumulate(opname, dacc, dcodes, scratch.meta, nxt)
    assert bits(dcodes) == bits(codes)
    assert bits(dacc) == bits(want)
    # fused range of the result == numpy min/max of it
    k = nxt.cpu().numpy().view(np.uint32)

    def dec(key):
        key = int(key)
        b = (key & 0x7FFFFFFF) if key & 0x80000000 else (~key & 0xFFFFFFFF)
        return np.array([b], np.uint32).view(np.float32)[0]

    assert dec(~int(k[0]) & 0xFFFFFFFF) == want.min()
    assert dec(k[1]) == want.max()
    assert k[2] == 0 and k[3] == 1


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_accumulate_large_random(dt):
    from paper_2505_14065_b200 import accumulate

    rng = np.random.default_rng(3)
    n = (1 << 24) + 5
    a = rng.normal(0, 1, n).astype(dt)
    b = rng.normal(0, 1, n).astype(dt)
    want = a + b
    da, db = to_dev(a), to_dev(b)
    accumulate("sum", da, db)
    assert bits(da) == bits(want)

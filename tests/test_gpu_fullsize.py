"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Each configuration C2..C5 is generated at full size, aligned on the GPU in one call
with device-resident inputs (as bench.py does), and a deterministic sample of pairs is
compared field by field with the oracle (which computes them one by one).  Every pair
is also checked against properties that hold at any size.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SAMPLE = 24


@pytest.fixture(scope="module")
def ctx(gpu_lib):
    c = gpu_lib.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5", "LS10"])
def test_full_size_sampled_parity(gpu_lib, ctx, name):
    import torch

    cfg = synth.CONFIGS[name]
    pairs = synth.generate(cfg)
    params = vars(cfg.scoring)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_ref, d_qry = dev(pairs.ref), dev(pairs.qry)
    d_roff, d_qoff = dev(pairs.ref_off.view(np.int64)), dev(pairs.qry_off.view(np.int64))
    out = torch.zeros(24 * pairs.n_pairs, dtype=torch.uint8, device="cuda")
    gpu_lib.align_batch(ctx, d_ref, d_roff, d_qry, d_qoff, params, out=out)
    assert ctx.stats()["packed16"] == 1
    got = gpu_lib.device_results(out)
    del d_ref, d_qry

    # properties of every pair
    m = np.diff(pairs.ref_off.astype(np.int64))
    n = np.diff(pairs.qry_off.astype(np.int64))
    term = got["zdrop_antidiag"]
    assert np.all((term == -1) | ((term >= 2) & (term < m + n)))           # Eq. 4: c < m+n
    assert np.all((got["ref_end"] >= 1) & (got["ref_end"] <= m))
    assert np.all((got["query_end"] >= 1) & (got["query_end"] <= n))
    d = got["ref_end"] - got["query_end"]
    assert np.all((d >= -params["band_left"]) & (d <= params["band_right"]))  # in band
    assert np.all(got["score"] <= params["match"] * np.minimum(got["ref_end"], got["query_end"]))
    nominal = np.array([oracle.nominal_cells(int(a), int(b), params["band_left"], params["band_right"])
                        for a, b in zip(m[:2000], n[:2000])])
    assert np.all(got["cells"][:2000] <= nominal)
    assert np.all(got["cells"][:2000][term[:2000] < 0] == nominal[term[:2000] < 0])

    # slot tiers: each pair at the narrowest front holding its clipped band
    D = np.minimum(params["band_left"], n) + np.minimum(params["band_right"], m) + 1
    tier = np.where(D > 512, 0, np.where(D > 256, 1, 2))
    assert ctx.stats()["tier_pairs"] == [int((tier == t).sum()) for t in range(3)]

    # sampled exact parity: evenly spaced pairs plus a few of every tier present
    idx = np.linspace(0, pairs.n_pairs - 1, SAMPLE).astype(np.int64)
    for t in range(3):
        idx = np.concatenate([idx, np.nonzero(tier == t)[0][:6]])
    rc, exp, _ = oracle.align_batch(pairs.subset(idx), params)
    assert rc == 0
    bad = np.nonzero(got[idx] != exp)[0]
    assert len(bad) == 0, f"{name}: pair {idx[bad[0]]} gpu={got[idx[bad[0]]]} oracle={exp[bad[0]]}"
    if name == "C3":
        assert (term >= 0).mean() > 0.2  # the Z-drop-heavy configuration really terminates
        # host inputs stream in chunks under the kernel, the late chunks
        # dispatched as one longest-first group: the same bytes as the device-input run
        host = gpu_lib.align_pairs(ctx, pairs, params)
        st = ctx.stats()
        assert st["input_chunks"] > 2 and 1 <= st["lpt_from_chunk"] < st["input_chunks"], st
        assert host.tobytes() == got.tobytes()

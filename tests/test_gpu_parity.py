"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Every comparison is on all five result fields (score, ref_end, query_end,
zdrop_antidiag, cells) for every pair: the path is integer work, so the bar is exact
equality (tests follow SURVEY.md §4 T5/T6/T7).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

SCORING = dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2)


@pytest.fixture(scope="module")
def ctx(gpu_lib):
    c = gpu_lib.Context(0)
    yield c
    c.close()


@pytest.fixture(params=["auto", "force32"])
def kflags(request, gpu_lib):
    """Run a test through the default kernel choice (the 16-bit packed kernel whenever it is
    exact for the parameters) and through the 32-bit kernel."""
    return 0 if request.param == "auto" else gpu_lib.FORCE_32BIT


def compare(gpu_lib, ctx, pairs, params, flags=0, **kw):
    got = gpu_lib.align_pairs(ctx, pairs, params, flags=flags, **kw)
    rc, exp, _ = oracle.align_batch(pairs, params)
    assert rc == 0
    bad = np.nonzero(got != exp)[0]
    if len(bad):
        k = int(bad[0])
        R, Q = pairs.pair(k)
        raise AssertionError(f"{len(bad)}/{len(got)} differ; pair {k} (m={len(R)}, n={len(Q)}) "
                             f"gpu={got[k]} oracle={exp[k]} params={params}")
    return got


def test_golden_cases_on_gpu(gpu_lib, ctx):
    from test_oracle import GOLDEN
    for R, Q, params, expected, cite in GOLDEN:
        got = gpu_lib.align_pairs(ctx, synth.from_list([(R, Q)]), params)
        assert tuple(got[0].tolist()) == expected, cite


@pytest.mark.parametrize("band", [0, 1, 2, 5, 16, 31, 32, 63, 64, 100, 255, 256, 300, 511])
def test_random_short_pairs(gpu_lib, ctx, kflags, band):
    rng = np.random.default_rng(1000 + band)
    pairs = synth.random_short_pairs(rng, 300, 400)
    for z in (-1, 0, 7, 40):
        compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=band, band_right=band, zdrop=z), flags=kflags)


# Band sizes D = bl + br + 1 that put the 16-bit kernel's low padding off = (-D) mod NREG
# at every interesting value, for both NREG = 8 (D <= 512) and NREG = 16 (D <= 1024, the
# eight-cap kernel for off <= 8 and the sixteen-cap one above): DESIGN.md §6.1 "Layout".
@pytest.mark.parametrize("bl,br", [(256, 255), (255, 255), (250, 255), (249, 254), (100, 3),
                                   (504, 504), (503, 504), (500, 500), (300, 292), (511, 511),
                                   (511, 500), (0, 600), (600, 0), (264, 264),
                                   # NREG = 4 (the narrow slot tier, D <= 256): off = 0..3
                                   (127, 128), (127, 127), (126, 127), (126, 126), (64, 64),
                                   # slot-tier boundaries: D = 257 (NREG 8), 513 (NREG 16)
                                   (128, 128), (256, 256)])
def test_band_layouts_long_pairs(gpu_lib, ctx, bl, br):
    rng = np.random.default_rng(7000 + bl * 1000 + br)
    lst = []
    for k in range(48):
        m = int(rng.integers(700, 1400))
        a = "".join("ACGT"[x] for x in rng.integers(0, 4, m))
        q = list(a)
        for t in range(len(q)):
            if rng.random() < 0.03:
                q[t] = "ACGT"[int(rng.integers(0, 4))]
        q = "".join(q)
        if k % 3 == 1:  # an indel that moves the path towards a band edge
            x = int(rng.integers(100, 400))
            q = q[:x] + q[x + int(rng.integers(5, 60)):]
        if k % 3 == 2:
            x = int(rng.integers(100, 400))
            q = q[:x] + "".join("ACGT"[y] for y in rng.integers(0, 4, int(rng.integers(5, 60)))) + q[x:]
        lst.append((a, q))
    pairs = synth.from_list(lst)
    for z in (-1, 100):
        compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=bl, band_right=br, zdrop=z))
        assert ctx.stats()["packed16"] == 1


def _pin_stress_pairs(rng, bl, br, n_pairs=24):
    """Pairs for the pinned 32-slot front: half of them carry their true alignment on a
    diagonal just under the band (the dead padding slots see long match runs while the
    band cells mismatch: the fastest rise of the dead slots against the band, DESIGN.md
    §6.1 "Layout"), the rest are 3%-error pairs with indels, some with chimeric tails."""
    lst = []
    for k in range(n_pairs):
        m = int(rng.integers(1500, 2600))
        a = "".join("ACGT"[x] for x in rng.integers(0, 4, m))
        if k % 2 == 0:  # Q = R shifted: matches on diagonal d = i - j = -(bl + s), under the band
            s = int(rng.integers(1, 5))
            q = "".join("ACGT"[x] for x in rng.integers(0, 4, bl + s)) + a
        else:
            q = "".join(c if rng.random() > 0.03 else "ACGT"[int(rng.integers(0, 4))] for c in a)
            if k % 4 == 1:
                x = int(rng.integers(100, 600))
                q = q[:x] + q[x + int(rng.integers(5, 80)):]
            if k % 8 == 3:  # chimeric tail (Z-drop)
                cut = int(rng.integers(len(q) // 3, len(q)))
                q = q[:cut] + "".join("ACGT"[x] for x in rng.integers(0, 4, len(q) - cut))
        lst.append((a, q[: max(bl + br + 2, len(q) - int(rng.integers(0, 50)))]))
    return lst


@pytest.mark.parametrize("off", list(range(16)))
def test_pinned_front_every_offset(gpu_lib, ctx, off):
    """The pinned 32-slot front (one capped padding slot, the dead ones re-pinned at each
    re-centring) at every low padding off = (-D) mod 16: bit-exact with
    the oracle, with and without Z-drop, and the stats name the front that ran."""
    D = 1024 - off
    bl = (D - 1) // 2
    br = D - 1 - bl
    rng = np.random.default_rng(9100 + off)
    pairs = synth.from_list(_pin_stress_pairs(rng, bl, br))
    for z in (-1, 60):
        compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=bl, band_right=br, zdrop=z))
        st = ctx.stats()
        assert st["packed16"] == 1 and st["tier_pairs"][0] == pairs.n_pairs and st["pin_off"] == off, st


@pytest.mark.parametrize("off", list(range(8)))
def test_pinned_16slot_front_every_offset(gpu_lib, ctx, off):
    """The 16-slot front's pinned instantiation (paired layout, one capped padding slot) at
    every off = (-D) mod 8 with 256 < D <= 512: bit-exact with the oracle, with and without
    Z-drop, and the stats name it."""
    D = 512 - off
    bl = (D - 1) // 2
    br = D - 1 - bl
    rng = np.random.default_rng(9300 + off)
    pairs = synth.from_list(_pin_stress_pairs(rng, bl, br))
    for z in (-1, 60):
        compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=bl, band_right=br, zdrop=z))
        st = ctx.stats()
        assert st["tier_pairs"][1] == pairs.n_pairs and st["pin_off8"] == off, st


def test_pinned_front_fast_rising_padding(gpu_lib, ctx):
    """Scoring with about the largest S + 2 alpha the 16-bit guard admits at D = 1001 (23) under a
    band whose padding diagonals match everywhere (the dead slots' fastest rise): the
    pinned front still matches the oracle; a mixed-off batch runs the capped front."""
    rng = np.random.default_rng(9200)
    lst = _pin_stress_pairs(rng, 500, 500, 16)
    pairs = synth.from_list(lst)
    for sc in (dict(match=1, mismatch=1, ambig=1, gap_open=11, gap_extend=2),
               dict(match=2, mismatch=4, ambig=4, gap_open=8, gap_extend=1)):
        compare(gpu_lib, ctx, pairs, dict(sc, band_left=500, band_right=500, zdrop=-1))
        st = ctx.stats()
        assert st["packed16"] == 1 and st["pin_off"] == 7, (sc, st)
    mixed = synth.from_list(lst[:8] + [(a, q[:400 + 7 * k]) for k, (a, q) in enumerate(lst[8:])])
    compare(gpu_lib, ctx, mixed, dict(SCORING, band_left=500, band_right=500, zdrop=100))
    assert ctx.stats()["pin_off"] == -1


def test_asymmetric_bands_and_penalties(gpu_lib, ctx, kflags):
    rng = np.random.default_rng(77)
    pairs = synth.random_short_pairs(rng, 200, 300)
    for bl, br in [(0, 7), (7, 0), (3, 60), (200, 17), (500, 500), (-1, 9), (9, -1)]:
        for (a, b, n, go, ge) in [(2, 4, 4, 4, 2), (1, 3, 1, 6, 2), (3, 5, 0, 7, 7), (2, 4, 4, 0, 0)]:
            compare(gpu_lib, ctx, pairs, dict(match=a, mismatch=b, ambig=n, gap_open=go,
                                              gap_extend=ge, band_left=bl, band_right=br, zdrop=25),
                    flags=kflags)


def test_unbounded_band_short_pairs(gpu_lib, ctx, kflags):
    rng = np.random.default_rng(5)
    pairs = synth.random_short_pairs(rng, 100, 200)
    compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=-1, band_right=-1, zdrop=-1), flags=kflags)
    compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=-1, band_right=-1, zdrop=30), flags=kflags)


def test_edge_corpus(gpu_lib, ctx, kflags):
    lst = [("A", "A"), ("A", "T"), ("N", "N"), ("A", "ACGTACGT" * 10), ("ACGTACGT" * 10, "A"),
           ("A" * 700, "A" * 3), ("A" * 3, "A" * 700), ("N" * 300, "N" * 300),
           ("ACGT" * 200, "TGCA" * 200), ("A" * 1000, "A" * 1000), ("AC" * 500, "CA" * 500),
           ("ACGTTGCA" * 120, "ACGTTGCA" * 119 + "ACG"), ("acgtn" * 50, "ACGTN" * 50)]
    pairs = synth.from_list(lst)
    for bl, br in [(0, 0), (1, 1), (3, 2), (100, 100), (511, 511), (0, 511), (511, 0)]:
        for z in (-1, 0, 5, 100):
            compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=bl, band_right=br, zdrop=z), flags=kflags)


def test_tie_heavy_corpus(gpu_lib, ctx, kflags):
    """Poly-A, dinucleotide and tandem repeats: many equal local maxima (readings R5/R6)."""
    rng = np.random.default_rng(11)
    lst = []
    for _ in range(150):
        unit = "".join(rng.choice(list("ACGT"), int(rng.integers(1, 6))))
        L = int(rng.integers(20, 600))
        R = (unit * (L // len(unit) + 1))[:L]
        Q = (unit * (L // len(unit) + 2))[int(rng.integers(0, 3)):][: int(rng.integers(10, L + 30))]
        if rng.random() < 0.5:  # break the repeat so Z-drop fires
            cut = int(rng.integers(1, len(Q)))
            Q = Q[:cut] + "".join(rng.choice(list("ACGT"), len(Q) - cut))
        lst.append((R, Q))
    pairs = synth.from_list(lst)
    for w in (3, 20, 100):
        for z in (0, 10, 50):
            compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=w, band_right=w, zdrop=z), flags=kflags)


def test_config_c1_full(gpu_lib, ctx, kflags):
    cfg = synth.CONFIGS["C1"]
    pairs = synth.generate(cfg)
    got = compare(gpu_lib, ctx, pairs, vars(cfg.scoring), flags=kflags)
    assert (got["zdrop_antidiag"] >= 0).sum() > 30  # Z-drop really exercised
    # the minimap2 q+e mapping (alpha=6, beta=2) as a second parity pass
    compare(gpu_lib, ctx, pairs, dict(vars(cfg.scoring), gap_open=6), flags=kflags)


def test_config_c0(gpu_lib, ctx, kflags):
    cfg = synth.CONFIGS["C0"]
    pairs = synth.generate(cfg, 0, 3000)
    rng = np.random.default_rng(0)
    for _ in range(4):
        w = int(rng.integers(0, 65))
        z = int(rng.integers(-1, 51))
        compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=w, band_right=w, zdrop=z), flags=kflags)


@pytest.mark.parametrize("name,k0,k1", [("C2", 0, 64), ("C3", 0, 24), ("C4", 0, 400), ("C5", 0, 40)])
def test_config_subsets(gpu_lib, ctx, kflags, name, k0, k1):
    """Pairs of the large configs, shapes as generated (full lengths), vs the oracle."""
    cfg = synth.CONFIGS[name]
    pairs = synth.generate(cfg, k0, k1)
    compare(gpu_lib, ctx, pairs, vars(cfg.scoring), flags=kflags)


def _tier(m, n, bl, br):
    """Slot tier of a pair (DESIGN.md §6.1 "Slot tiers"): 0, 1, 2 for a 32-lane front of
    32, 16, 8 slots per lane, the narrowest that holds the pair's D clipped diagonals."""
    D = min(bl, n) + min(br, m) + 1
    return 0 if D > 512 else (1 if D > 256 else 2)


def test_slot_tiers_mixed_batch(gpu_lib, ctx):
    """A batch whose pairs need all three slot tiers (w = 500; short pairs clip the band):
    every tier launch is bit-exact, the per-tier counts match the pairs' D, and one launch
    at the widest front (SINGLE_TIER) or input order gives the same bytes."""
    rng = np.random.default_rng(4242)
    lst = []
    for k in range(240):
        L = int([rng.integers(20, 120), rng.integers(130, 250), rng.integers(300, 1500)][k % 3])
        a = "".join("ACGT"[x] for x in rng.integers(0, 4, L))
        q = "".join(c if rng.random() > 0.04 else "ACGT"[int(rng.integers(0, 4))] for c in a)
        if k % 5 == 0:  # chimeric tail: Z-drop fires
            cut = int(rng.integers(1, len(q)))
            q = q[:cut] + "".join("ACGT"[x] for x in rng.integers(0, 4, len(q) - cut))
        lst.append((a, q[: int(rng.integers(max(1, len(q) // 2), len(q) + 1))]))
    pairs = synth.from_list(lst)
    params = dict(SCORING, band_left=500, band_right=500, zdrop=60)
    got = compare(gpu_lib, ctx, pairs, params)
    want = [0, 0, 0]
    for R, Q in lst:
        want[_tier(len(R), len(Q), 500, 500)] += 1
    assert min(want) > 0
    st = ctx.stats()
    assert st["packed16"] == 1 and st["tier_pairs"] == want, (st, want)
    assert st["kernel_launches"] == 1 + 3  # prep + one align launch per tier
    one = gpu_lib.align_pairs(ctx, pairs, params, flags=gpu_lib.SINGLE_TIER)
    assert ctx.stats()["tier_pairs"] == [len(lst), 0, 0]
    assert one.tobytes() == got.tobytes()
    inp = gpu_lib.align_pairs(ctx, pairs, params, flags=gpu_lib.ORDER_INPUT)
    assert inp.tobytes() == got.tobytes()
    # the no-refill ablation (static warp assignment) in both orders, and with the 32-bit
    # kernel, gives the same bytes
    for fl in (gpu_lib.STATIC_ASSIGN, gpu_lib.STATIC_ASSIGN | gpu_lib.ORDER_INPUT,
               gpu_lib.STATIC_ASSIGN | gpu_lib.FORCE_32BIT):
        st_ = gpu_lib.align_pairs(ctx, pairs, params, flags=fl)
        assert st_.tobytes() == got.tobytes(), fl
    # a batch that is all narrow runs the NREG = 4 front alone
    short = pairs.subset([k for k in range(len(lst)) if k % 3 == 0])
    compare(gpu_lib, ctx, short, params)
    assert ctx.stats()["tier_pairs"] == [0, 0, short.n_pairs] and ctx.stats()["slots_per_lane"] == 8


def test_streamed_host_chunks(gpu_lib, monkeypatch):
    """Host inputs stream in many small chunks (AGATHA_CHUNK_BYTES shrinks them) under the
    running kernel, warps waiting on per-chunk arrival flags, the late chunks dispatched as
    one longest-first group: identical bytes to the device-input run."""
    import torch
    monkeypatch.setenv("AGATHA_CHUNK_BYTES", "262144")
    c = gpu_lib.Context(0)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for name, k1, grouped in (("C2", 200, True), ("C1", 1000, False)):
        cfg = synth.CONFIGS[name]
        pairs = synth.generate(cfg, 0, k1)
        params = vars(cfg.scoring)
        host = gpu_lib.align_pairs(c, pairs, params)
        st = c.stats()
        assert st["input_chunks"] > 4, st
        # w = 500 is compute-bound (late chunks grouped); C1's w = 100 is copy-bound
        assert (st["lpt_from_chunk"] < st["input_chunks"]) == grouped, st
        out = torch.zeros(24 * pairs.n_pairs, dtype=torch.uint8, device="cuda")
        gpu_lib.align_batch(c, dev(pairs.ref), dev(pairs.ref_off.view(np.int64)), dev(pairs.qry),
                            dev(pairs.qry_off.view(np.int64)), params, out=out)
        assert gpu_lib.device_results(out).tobytes() == host.tobytes()
        idx = np.arange(0, pairs.n_pairs, max(1, pairs.n_pairs // 12))
        rc, exp, _ = oracle.align_batch(pairs.subset(idx), params)
        assert rc == 0 and host[idx].tobytes() == exp.tobytes()
    c.close()


def test_kernel_selection(gpu_lib, ctx):
    """The 16-bit packed kernel runs for the paper's scoring at w = 500; parameters outside
    its exactness guard run the 32-bit kernel."""
    pairs = synth.generate(synth.CONFIGS["C2"], 0, 8)
    gpu_lib.align_pairs(ctx, pairs, vars(synth.CONFIGS["C2"].scoring))
    assert ctx.stats()["packed16"] == 1
    gpu_lib.align_pairs(ctx, pairs, vars(synth.CONFIGS["C2"].scoring), flags=gpu_lib.FORCE_32BIT)
    assert ctx.stats()["packed16"] == 0
    big = dict(SCORING, match=40, band_left=500, band_right=500, zdrop=400)
    compare(gpu_lib, ctx, pairs, big)
    assert ctx.stats()["packed16"] == 0


def test_ordering_invariance(gpu_lib, ctx):
    """Dispatch order (longest-first queue vs input order) never changes a result."""
    cfg = synth.CONFIGS["C1"]
    pairs = synth.generate(cfg, 0, 300)
    a = gpu_lib.align_pairs(ctx, pairs, vars(cfg.scoring))
    b = gpu_lib.align_pairs(ctx, pairs, vars(cfg.scoring), flags=gpu_lib.ORDER_INPUT)
    assert a.tobytes() == b.tobytes()
    # and a pair's result does not depend on its batch mates
    c = gpu_lib.align_pairs(ctx, pairs.subset([7, 3, 250]), vars(cfg.scoring))
    assert c.tobytes() == a[[7, 3, 250]].tobytes()


def test_device_buffers_and_stream(gpu_lib, ctx):
    import torch
    cfg = synth.CONFIGS["C1"]
    pairs = synth.generate(cfg, 0, 200)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = torch.zeros(24 * pairs.n_pairs, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gpu_lib.align_batch(ctx, dev(pairs.ref), dev(pairs.ref_off.view(np.int64)), dev(pairs.qry),
                            dev(pairs.qry_off.view(np.int64)), vars(cfg.scoring), out=out, stream=s)
    got = gpu_lib.device_results(out)
    rc, exp, _ = oracle.align_batch(pairs, vars(cfg.scoring))
    assert got.tobytes() == exp.tobytes()


def test_localmax_trace_matches_oracle(gpu_lib, ctx, kflags):
    cfg = synth.CONFIGS["C1"]
    pairs = synth.generate(cfg, 40, 60)
    params = vars(cfg.scoring)
    for k in range(pairs.n_pairs):
        R, Q = pairs.pair(k)
        cap = len(R) + len(Q) + 1
        gs, gi = gpu_lib.localmax_trace(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off,
                                        params, k, cap, flags=kflags)
        rc, res, (os_, oi) = oracle.align_one(R, Q, params, trace=True)
        c_end = res[3] if res[3] >= 0 else len(R) + len(Q)
        reached = np.arange(cap) <= c_end
        assert np.array_equal(gi[reached], oi[reached]), k
        nonempty = reached & (oi >= 0)
        assert np.array_equal(gs[nonempty], os_[nonempty]), k


def test_pack4_matches_oracle(gpu_lib, ctx):
    import torch
    rng = np.random.default_rng(3)
    for L in (1, 7, 8, 9, 63, 64, 65, 1000, 12345):
        s = rng.choice(np.frombuffer(b"ACGTNacgtn", np.uint8), L).tobytes()
        dev = torch.from_numpy(np.frombuffer(s, np.uint8).copy()).cuda()
        for rev in (False, True):
            words = torch.zeros((L + 7) // 8, dtype=torch.int32, device="cuda")
            rc = gpu_lib.pack4(ctx, dev, words, flags=gpu_lib.PACK_REVERSE if rev else 0)
            assert rc == 0
            orc, exp = oracle.pack4(s, reverse=rev)
            assert np.array_equal(words.cpu().numpy().view(np.uint32), exp)
    bad = torch.from_numpy(np.frombuffer(b"ACGTXACG", np.uint8).copy()).cuda()
    words = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert gpu_lib.pack4(ctx, bad, words) == gpu_lib.ECHAR
    assert gpu_lib.pack4(ctx, bad, words, flags=gpu_lib.N_MAP) == 0
    assert words.cpu().numpy().view(np.uint32)[0] == oracle.pack4(b"ACGTXACG", n_map=True)[1][0]


def test_plan_matches_oracle(gpu_lib, ctx):
    import torch
    cfg = synth.CONFIGS["C4"]
    pairs = synth.generate(cfg, 0, 2000)
    params = vars(cfg.scoring)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    order = torch.zeros(pairs.n_pairs, dtype=torch.int32, device="cuda")
    nominal = torch.zeros(pairs.n_pairs, dtype=torch.int32, device="cuda")
    gpu_lib.plan(ctx, dev(pairs.ref), dev(pairs.ref_off.view(np.int64)), dev(pairs.qry),
                 dev(pairs.qry_off.view(np.int64)), params, order, nominal)
    nom = nominal.cpu().numpy().view(np.uint32).astype(np.int64)
    ordr = order.cpu().numpy().view(np.uint32).astype(np.int64)
    rl = np.diff(pairs.ref_off.astype(np.int64))
    ql = np.diff(pairs.qry_off.astype(np.int64))
    exp = np.array([oracle.nominal_cells(int(m), int(n), 500, 500) for m, n in zip(rl, ql)])
    assert np.array_equal(nom, exp)
    assert sorted(ordr.tolist()) == list(range(pairs.n_pairs))      # a permutation
    assert np.all(np.diff(nom[ordr]) <= 0)                            # longest first


def test_error_codes(gpu_lib, ctx):
    ok = synth.from_list([("ACGT", "ACGT")])
    with pytest.raises(gpu_lib.AgathaError) as e:
        gpu_lib.align_pairs(ctx, synth.from_list([("ACGT", "AXGT")]), SCORING)
    assert e.value.code == gpu_lib.ECHAR
    got = gpu_lib.align_pairs(ctx, synth.from_list([("ACGT", "AXGT")]), SCORING, flags=gpu_lib.N_MAP)
    assert tuple(got[0].tolist())[:3] == oracle.align_one("ACGT", "ANGT", SCORING)[1][:3]
    with pytest.raises(gpu_lib.AgathaError) as e:
        gpu_lib.align_pairs(ctx, synth.from_list([("ACGT", "")]), SCORING)
    assert e.value.code == gpu_lib.EEMPTY
    with pytest.raises(gpu_lib.AgathaError) as e:
        gpu_lib.align_pairs(ctx, synth.from_list([]), SCORING)
    assert e.value.code == gpu_lib.EEMPTY
    for bad in (dict(match=0), dict(mismatch=-1), dict(gap_open=1, gap_extend=2), dict(ambig=-2)):
        with pytest.raises(gpu_lib.AgathaError) as e:
            gpu_lib.align_pairs(ctx, ok, dict(SCORING, **bad))
        assert e.value.code == gpu_lib.EINVAL
    with pytest.raises(gpu_lib.AgathaError) as e:  # wider than 4096 diagonals
        gpu_lib.align_pairs(ctx, synth.from_list([("A" * 5000, "A" * 5000)]),
                            dict(SCORING, band_left=2048, band_right=2048))
    assert e.value.code == gpu_lib.ERANGE
    with pytest.raises(gpu_lib.AgathaError) as e:  # penalty beyond the int8 score table
        gpu_lib.align_pairs(ctx, ok, dict(SCORING, mismatch=200))
    assert e.value.code == gpu_lib.ERANGE


@pytest.mark.parametrize("w", [500, 200, 100])
def test_bad_base_beyond_the_band(gpu_lib, ctx, kflags, w):
    """A non-ACGTN byte is refused wherever it sits, also where the band never reaches
    (very unequal lengths: R bases past n + w, Q bases past m + w), on every front; with
    N_MAP it reads as N, exactly as in the oracle (R17)."""
    rng = np.random.default_rng(5000 + w)
    a = "".join("ACGT"[x] for x in rng.integers(0, 4, 20000))
    b = "".join("ACGT"[x] for x in rng.integers(0, 4, 1200))
    for R, Q in ((a[:19000] + "X" + a[19001:], b), (b, a[:19500] + "x" + a[19501:])):
        pairs = synth.from_list([(R, Q), (a[:3000], a[5:3000])])
        params = dict(SCORING, band_left=w, band_right=w, zdrop=-1)
        with pytest.raises(gpu_lib.AgathaError) as e:
            gpu_lib.align_pairs(ctx, pairs, params, flags=kflags)
        assert e.value.code == gpu_lib.ECHAR
        got = gpu_lib.align_pairs(ctx, pairs, params, flags=kflags | gpu_lib.N_MAP)
        mapped = synth.from_list([(R.replace("X", "N"), Q.replace("x", "N")), (a[:3000], a[5:3000])])
        rc, exp, _ = oracle.align_batch(mapped, params)
        assert rc == 0 and got.tobytes() == exp.tobytes()


def test_variant_golden_on_gpu(gpu_lib, ctx, kflags):
    from test_oracle import VARIANTS
    for R, Q, params, expected, cite in VARIANTS:
        got = gpu_lib.align_pairs(ctx, synth.from_list([(R, Q)]), dict(SCORING, **params), flags=kflags)
        assert tuple(got[0].tolist()) == expected, cite


@pytest.mark.parametrize("variant", [1, 2, 4, 7])
def test_variants_random_and_c1(gpu_lib, ctx, kflags, variant):
    rng = np.random.default_rng(900 + variant)
    pairs = synth.random_short_pairs(rng, 200, 300)
    for w, z in [(5, 0), (32, 20), (300, 40), (-1, 10)]:
        compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=w, band_right=w, zdrop=z, variant=variant),
                flags=kflags)
    cfg = synth.CONFIGS["C1"]
    compare(gpu_lib, ctx, synth.generate(cfg, 0, 300), dict(vars(cfg.scoring), variant=variant),
            flags=kflags)


# NEXT #3, the wide-band tier: bands of more than 1024 diagonals run the 32-bit kernel
# with two (D <= 2048) or four (D <= 4096) warps per pair (DESIGN.md §6.1 "Wide bands").
@pytest.mark.parametrize("bl,br,warps", [(512, 512, 2), (700, 400, 2), (1023, 1024, 2),
                                         (1024, 1024, 4), (1500, 900, 4), (2047, 2048, 4),
                                         (0, 1100, 2), (3000, 1000, 4)])
def test_wide_bands(gpu_lib, ctx, bl, br, warps):
    rng = np.random.default_rng(9000 + bl + 7 * br)
    lst = []
    for k in range(24):
        m = int(rng.integers(1500, 4500))
        a = "".join("ACGT"[x] for x in rng.integers(0, 4, m))
        q = list(a)
        for t in range(len(q)):
            if rng.random() < 0.05:
                q[t] = "ACGT"[int(rng.integers(0, 4))]
        q = "".join(q)
        if k % 4 == 1:  # a long indel: the optimum leaves the main diagonal by hundreds
            x = int(rng.integers(200, 800))
            q = q[:x] + q[x + int(rng.integers(200, 900)):]
        if k % 4 == 2:
            x = int(rng.integers(200, 800))
            q = q[:x] + "".join("ACGT"[y] for y in rng.integers(0, 4, int(rng.integers(200, 900)))) + q[x:]
        if k % 4 == 3:  # chimeric tail (Z-drop)
            x = int(rng.integers(500, len(q)))
            q = q[:x] + "".join("ACGT"[y] for y in rng.integers(0, 4, len(q) - x))
        lst.append((a, q))
    lst += [("ACGT" * 600, "A"), ("A", "ACGT" * 700), ("N" * 1500, "N" * 2600)]
    pairs = synth.from_list(lst)
    for z in (-1, 150):
        compare(gpu_lib, ctx, pairs, dict(SCORING, band_left=bl, band_right=br, zdrop=z))
        st = ctx.stats()
        # the widest band actually used decides the tier
        assert st["packed16"] == 0 and st["warps_per_pair"] == warps, st


def test_wide_band_trace(gpu_lib, ctx):
    """Eq. 5 trace of one pair through the four-warp tier equals the oracle's."""
    rng = np.random.default_rng(77)
    a = "".join("ACGT"[x] for x in rng.integers(0, 4, 3000))
    q = a[:1400] + a[1800:] + "".join("ACGT"[x] for x in rng.integers(0, 4, 300))
    pairs = synth.from_list([(a, q), (a[:2000], a[100:2500])])
    params = dict(SCORING, band_left=1600, band_right=1700, zdrop=200)
    for k in range(pairs.n_pairs):
        R, Q = pairs.pair(k)
        cap = len(R) + len(Q) + 1
        gs, gi = gpu_lib.localmax_trace(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off,
                                        params, k, cap)
        assert ctx.stats()["warps_per_pair"] == 4
        rc, res, (os_, oi) = oracle.align_one(R, Q, params, trace=True)
        assert rc == 0
        c_end = res[3] if res[3] >= 0 else len(R) + len(Q)
        reached = np.arange(cap) <= c_end
        assert np.array_equal(gi[reached], oi[reached]), k
        nonempty = reached & (oi >= 0)
        assert np.array_equal(gs[nonempty], os_[nonempty]), k


# NEXT #1, cross-GPU dynamic balancing: participants that share one pair counter align
# disjoint subsets of the same batch; their merged rows equal the ORACLE's (and the
# one-context GPU run), and each slot tier's pairs are claimed from that tier's counter.
def _merge_rows(*outs):
    acc = np.zeros(len(outs[0]) * 3, np.int64)
    for o in outs:
        acc += o.view(np.int64)
    return acc.view(oracle.RESULT_DTYPE)


def _tiers(pairs, params):
    """Slot tier of each pair: the narrowest 32-lane front holding its
    clipped band D = min(bl, n) + min(br, m) + 1."""
    m = np.diff(pairs.ref_off).astype(np.int64)
    n = np.diff(pairs.qry_off).astype(np.int64)
    bl = np.where(params["band_left"] < 0, n, np.minimum(params["band_left"], n))
    br = np.where(params["band_right"] < 0, m, np.minimum(params["band_right"], m))
    D = bl + br + 1
    return np.where(D > 512, 0, np.where(D > 256, 1, 2))


def _check_claims(outs, pairs, params, exp):
    claimed = [o["cells"] != 0 for o in outs]
    assert not np.any(claimed[0] & claimed[1]), "a pair was aligned twice"
    assert np.all(claimed[0] | claimed[1]), "a pair was never aligned"
    tiers = _tiers(pairs, params)
    for t in range(3):
        in_t = tiers == t
        assert sum(int((c & in_t).sum()) for c in claimed) == int(in_t.sum()), t
    merged = _merge_rows(*outs)
    bad = np.nonzero(merged != exp)[0]
    assert len(bad) == 0, (len(bad), int(bad[0]), merged[bad[0]], exp[bad[0]])
    return merged


@pytest.mark.parametrize("name", ["C5", "LS10"])  # LS10: two slot tiers, one counter each
def test_shared_queue_two_contexts(gpu_lib, ctx, name):
    import threading
    import torch
    cfg = synth.CONFIGS[name]
    pairs = synth.generate(cfg, 0, 600)
    params = vars(cfg.scoring)
    rc, exp, _ = oracle.align_batch(pairs, params)
    assert rc == 0
    if name == "LS10":
        assert len(set(_tiers(pairs, params).tolist())) == 2
    full = gpu_lib.align_pairs(ctx, pairs, params)
    assert full.tobytes() == exp.tobytes()
    c2 = gpu_lib.Context(0)
    q = gpu_lib.SharedQueue.create(ctx)
    try:
        for rep in range(3):
            q.reset()
            torch.cuda.synchronize()
            outs = [np.zeros(pairs.n_pairs, gpu_lib.RESULT_DTYPE) for _ in range(2)]
            errs = []

            def run(k, c):
                try:
                    s = torch.cuda.Stream()
                    gpu_lib.align_pairs_q(c, pairs, params, outs[k], q, s)
                except Exception as e:  # noqa: BLE001 -- surfaced below
                    errs.append(e)

            th = [threading.Thread(target=run, args=(k, c)) for k, c in enumerate((ctx, c2))]
            for t in th:
                t.start()
            for t in th:
                t.join()
            assert not errs, errs
            _check_claims(outs, pairs, params, exp)
    finally:
        q.close()
        c2.close()


def test_shared_queue_refuses_a_different_batch(gpu_lib, ctx):
    """a participant whose order would differ (another flag, another batch) is
    refused with EINVAL before it claims anything, instead of silently aligning some
    pairs twice and others never."""
    import torch
    cfg = synth.CONFIGS["LS10"]
    pairs = synth.generate(cfg, 0, 200)
    params = vars(cfg.scoring)
    q = gpu_lib.SharedQueue.create(ctx)
    c2 = gpu_lib.Context(0)
    try:
        q.reset()
        torch.cuda.synchronize()
        out = np.zeros(pairs.n_pairs, gpu_lib.RESULT_DTYPE)
        gpu_lib.align_pairs_q(ctx, pairs, params, out, q)
        out2 = np.zeros(pairs.n_pairs, gpu_lib.RESULT_DTYPE)
        with pytest.raises(gpu_lib.AgathaError) as ei:
            gpu_lib.align_pairs_q(c2, pairs, params, out2, q, flags=gpu_lib.SINGLE_TIER)
        assert ei.value.code == -1  # AGATHA_EINVAL
        other = synth.generate(cfg, 200, 400)
        with pytest.raises(gpu_lib.AgathaError):
            gpu_lib.align_pairs_q(c2, other, params, out2, q)
        assert not out2["cells"].any()  # refused before claiming
        # the same batch and flags is accepted (claims nothing: the queue is drained)
        gpu_lib.align_pairs_q(c2, pairs, params, out2, q)
        assert not out2["cells"].any()
        rc, exp, _ = oracle.align_batch(pairs, params)
        assert out.tobytes() == exp.tobytes()
        # after a reset the fingerprint is cleared: another batch is accepted
        q.reset()
        torch.cuda.synchronize()
        gpu_lib.align_pairs_q(c2, other, params, out2, q, flags=gpu_lib.SINGLE_TIER)
        rc, exp2, _ = oracle.align_batch(other, params)
        assert out2.tobytes() == exp2.tobytes()
    finally:
        c2.close()
        q.close()


def _ipc_worker(rank, handle_q, result_q, done_q):
    import torch
    from paper_2403_06478_b200 import agatha
    torch.cuda.set_device(0)
    c = agatha.Context(0)
    cfg = synth.CONFIGS["C5"]
    pairs = synth.generate(cfg, 0, 400)
    if rank == 0:
        q = agatha.SharedQueue.create(c)
        handle_q.put(q.handle)
    else:
        q = agatha.SharedQueue.open(c, handle_q.get())
    out = np.zeros(pairs.n_pairs, agatha.RESULT_DTYPE)
    result_q.put(("ready", rank))
    agatha.align_batch(c, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, vars(cfg.scoring),
                       out=out, queue=q)
    result_q.put((rank, out.tobytes()))
    if rank == 0:
        # the counter lives in rank 0's allocation: keep it until rank 1 is done with it
        done_q.get(timeout=300)
    else:
        q.close()
        done_q.put("done")
    if rank == 0:
        q.close()
    c.close()


def test_shared_queue_two_processes(gpu_lib, ctx):
    """The counter crosses processes through its CUDA IPC handle (agatha_queue_open),
    as it would cross GPUs; claims use system-scope atomics."""
    import torch.multiprocessing as tmp
    mpc = tmp.get_context("spawn")
    hq, rq, dq = mpc.Queue(), mpc.Queue(), mpc.Queue()
    ps = [mpc.Process(target=_ipc_worker, args=(r, hq, rq, dq)) for r in range(2)]
    for p_ in ps:
        p_.start()
    got = {}
    while len(got) < 2:
        item = rq.get(timeout=300)
        if item[0] != "ready":
            got[item[0]] = np.frombuffer(item[1], gpu_lib.RESULT_DTYPE)
    for p_ in ps:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    cfg = synth.CONFIGS["C5"]
    pairs = synth.generate(cfg, 0, 400)
    params = vars(cfg.scoring)
    rc, exp, _ = oracle.align_batch(pairs, params)
    assert rc == 0
    _check_claims([got[0], got[1]], pairs, params, exp)


# NEXT #1 without replicated inputs: a federated batch is the
# concatenation of several owners' device batches; a claimed pair's inputs are read from
# its owner's memory (another process's, or over NVLink another GPU's).
def _dev_owner(pairs):
    import torch
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return (dev(pairs.ref), dev(pairs.ref_off.view(np.int64)), dev(pairs.qry), dev(pairs.qry_off.view(np.int64)))


@pytest.mark.parametrize("name", ["C5", "LS10", "C1"])
def test_federated_owners_one_context(gpu_lib, ctx, name):
    import torch
    cfg = synth.CONFIGS[name]
    cuts = [0, 70, 71, 300]  # owners of 70, 1 and 229 pairs
    parts = [synth.generate(cfg, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    whole = synth.generate(cfg, 0, cuts[-1])
    params = vars(cfg.scoring)
    rc, exp, _ = oracle.align_batch(whole, params)
    assert rc == 0
    owners = [_dev_owner(p) for p in parts]
    for flags in (0, gpu_lib.SINGLE_TIER, gpu_lib.FORCE_32BIT, gpu_lib.ORDER_INPUT):
        out = torch.zeros(24 * whole.n_pairs, dtype=torch.uint8, device="cuda")
        gpu_lib.align_federated(ctx, owners, params, out, flags=flags)
        got = gpu_lib.device_results(out)
        bad = np.nonzero(got != exp)[0]
        assert len(bad) == 0, (flags, len(bad), int(bad[0]), got[bad[0]], exp[bad[0]])


def _fed_worker(rank, handle_q, result_q, done_q):
    """One participant: it owns pairs [200 rank, 200 rank + 200) of C5 in its own IPC
    buffers (its H2D is its own shard), maps the other's, and claims from one queue."""
    import torch
    from paper_2403_06478_b200 import agatha
    torch.cuda.set_device(0)
    c = agatha.Context(0)
    cfg = synth.CONFIGS["C5"]
    mine = synth.generate(cfg, 200 * rank, 200 * rank + 200)
    arrays = [mine.ref, mine.ref_off.view(np.uint8), mine.qry, mine.qry_off.view(np.uint8)]
    bufs = []
    for a in arrays:
        b = agatha.IpcBuffer.alloc(c, a.nbytes)
        b.copy_from_host(a)  # H2D: this participant copies only its own shard
        bufs.append(b)
    q = agatha.SharedQueue.create(c) if rank == 0 else None
    handle_q.put((rank, [b.handle for b in bufs], [a.nbytes for a in arrays], q.handle if q else None))
    peers = {}
    while len(peers) < 1:
        item = handle_q.get(timeout=300)
        if item[0] == rank:  # own message came back: put it back for the other one
            handle_q.put(item)
            import time
            time.sleep(0.05)
            continue
        peers[item[0]] = item
    other = peers[1 - rank]
    if rank == 1:
        q = agatha.SharedQueue.open(c, other[3])
    ob = [agatha.IpcBuffer.open(c, h, n) for h, n in zip(other[1], other[2])]

    def owner(bs, npairs):
        return (agatha.DevicePtr(bs[0].ptr, bs[0].nbytes), agatha.DevicePtr(bs[1].ptr, npairs + 1),
                agatha.DevicePtr(bs[2].ptr, bs[2].nbytes), agatha.DevicePtr(bs[3].ptr, npairs + 1))

    owners = [owner(bufs, 200), owner(ob, 200)] if rank == 0 else [owner(ob, 200), owner(bufs, 200)]
    out = torch.zeros(24 * 400, dtype=torch.uint8, device="cuda")
    result_q.put(("ready", rank))
    agatha.align_federated(c, owners, vars(cfg.scoring), out, queue=q)
    torch.cuda.synchronize()
    result_q.put((rank, out.cpu().numpy().tobytes()))
    # rank 0's queue and both processes' buffers are mapped by the other: close only
    # after both are done
    done_q.put(rank)
    seen = {rank}
    while len(seen) < 2:
        r = done_q.get(timeout=300)
        if r in seen:
            done_q.put(r)
            import time
            time.sleep(0.05)
        seen.add(r)
    for b in ob:
        b.close()
    if rank == 1:
        q.close()
    import time
    time.sleep(1.0)
    for b in bufs:
        b.close()
    if rank == 0:
        q.close()
    c.close()


def test_federated_two_processes_shared_queue(gpu_lib, ctx):
    import torch.multiprocessing as tmp
    mpc = tmp.get_context("spawn")
    hq, rq, dq = mpc.Queue(), mpc.Queue(), mpc.Queue()
    ps = [mpc.Process(target=_fed_worker, args=(r, hq, rq, dq)) for r in range(2)]
    for p_ in ps:
        p_.start()
    got = {}
    while len(got) < 2:
        item = rq.get(timeout=300)
        if item[0] != "ready":
            got[item[0]] = np.frombuffer(item[1], gpu_lib.RESULT_DTYPE)
    for p_ in ps:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    cfg = synth.CONFIGS["C5"]
    whole = synth.generate(cfg, 0, 400)
    params = vars(cfg.scoring)
    rc, exp, _ = oracle.align_batch(whole, params)
    assert rc == 0
    _check_claims([got[0], got[1]], whole, params, exp)


# NEXT #4: minimap2-style end scores (agatha_ends_t, reading R19) from every
# kernel (16-bit fronts of all slot tiers, 32-bit, wide tier) against the oracle.
def compare_ends(gpu_lib, ctx, pairs, params, flags=0):
    got, gends = gpu_lib.align_pairs_ends(ctx, pairs, params, flags=flags)
    rc, exp, eends, _ = oracle.align_batch_ends(pairs, params)
    assert rc == 0
    bad = np.nonzero(got != exp)[0]
    assert len(bad) == 0, (len(bad), int(bad[0]), got[bad[0]], exp[bad[0]])
    fields = ["mqe", "mqe_i", "mte", "mte_j", "end_score"]
    bad = np.nonzero(np.any(np.stack([gends[f] != eends[f] for f in fields]), axis=0))[0]
    if len(bad):
        k = int(bad[0])
        R, Q = pairs.pair(k)
        raise AssertionError(f"ends: {len(bad)}/{len(got)} differ; pair {k} (m={len(R)}, n={len(Q)}) "
                             f"gpu={gends[k]} oracle={eends[k]} params={params} flags={flags}")
    return gends


@pytest.mark.parametrize("band", [0, 1, 3, 16, 63, 200, 511])
def test_ends_random_short_pairs(gpu_lib, ctx, kflags, band):
    rng = np.random.default_rng(5000 + band)
    pairs = synth.random_short_pairs(rng, 200, 300)
    for z in (-1, 0, 9, 40):
        compare_ends(gpu_lib, ctx, pairs, dict(SCORING, band_left=band, band_right=band, zdrop=z), flags=kflags)
    compare_ends(gpu_lib, ctx, pairs, dict(SCORING, band_left=band, band_right=band // 2 + 3, zdrop=20,
                                           variant=7), flags=kflags)


@pytest.mark.parametrize("name", ["C1", "C3", "LS10"])
def test_ends_synthetic_configs(gpu_lib, ctx, kflags, name):
    cfg = synth.CONFIGS[name]
    n = {"C1": 400, "C3": 24, "LS10": 300}[name]
    pairs = synth.generate(cfg, 0, n)
    e = compare_ends(gpu_lib, ctx, pairs, vars(cfg.scoring), flags=kflags)
    assert (e["mqe"] != gpu_lib.NO_SCORE).sum() > 0


def test_ends_wide_tier_and_unbounded(gpu_lib, ctx):
    pairs = synth.generate(synth.CONFIGS["CW1"], 0, 6)
    pairs = synth.from_list([(R[:2500], Q[:2400]) for R, Q in (pairs.pair(k) for k in range(6))])
    for prm in (dict(SCORING, band_left=700, band_right=700, zdrop=400),
                dict(SCORING, band_left=1500, band_right=1600, zdrop=-1)):
        compare_ends(gpu_lib, ctx, pairs, prm)
        assert ctx.stats()["warps_per_pair"] > 1
    short = synth.random_short_pairs(np.random.default_rng(9), 120, 200)
    compare_ends(gpu_lib, ctx, short, dict(SCORING, band_left=-1, band_right=-1, zdrop=-1))

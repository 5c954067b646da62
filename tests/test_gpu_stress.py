"""Stress cases for the 16-bit packed kernel's exactness argument.

Each case is run through the default kernel (16-bit whenever the guard allows) and the
32-bit kernel, and both are compared with the oracle on every field:

* Z-drop off over long unrelated tails: the anti-diagonal max falls for thousands of
  anti-diagonals, so the base re-centring must follow it down;
* large indels that push the optimal path to the band edge and out of it;
* scoring at the edge of the guard (spread close to the 15000 limit);
* poly-N and all-mismatch stretches (the most negative scores);
* reads much longer than references and vice versa (long head/tail phases).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(gpu_lib):
    c = gpu_lib.Context(0)
    yield c
    c.close()


def both(gpu_lib, ctx, pairs, params, expect16=None):
    rc, exp, _ = oracle.align_batch(pairs, params)
    assert rc == 0
    for flags in (0, gpu_lib.FORCE_32BIT):
        got = gpu_lib.align_pairs(ctx, pairs, params, flags=flags)
        if flags == 0 and expect16 is not None:
            assert ctx.stats()["packed16"] == int(expect16)
        bad = np.nonzero(got != exp)[0]
        assert len(bad) == 0, (f"flags={flags}: pair {bad[0]} gpu={got[bad[0]]} "
                               f"oracle={exp[bad[0]]} params={params}")


def rand_seq(rng, n, alphabet="ACGT"):
    return "".join(rng.choice(list(alphabet), n))


def test_long_unrelated_tails_z_off(gpu_lib, ctx):
    rng = np.random.default_rng(21)
    lst = []
    for _ in range(24):
        head = rand_seq(rng, int(rng.integers(50, 2000)))
        lst.append((head + rand_seq(rng, int(rng.integers(3000, 9000))),
                    head + rand_seq(rng, int(rng.integers(3000, 9000)))))
    pairs = synth.from_list(lst)
    for w in (100, 500):
        both(gpu_lib, ctx, pairs, dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                                       band_left=w, band_right=w, zdrop=-1), expect16=True)


def test_large_indels(gpu_lib, ctx):
    rng = np.random.default_rng(22)
    lst = []
    for _ in range(30):
        a = rand_seq(rng, int(rng.integers(500, 3000)))
        b = rand_seq(rng, int(rng.integers(500, 3000)))
        ins = rand_seq(rng, int(rng.integers(100, 900)))
        if rng.random() < 0.5:
            lst.append((a + ins + b, a + b))  # deletion from the read
        else:
            lst.append((a + b, a + ins + b))  # insertion into the read
    pairs = synth.from_list(lst)
    for w, z in [(100, 400), (500, 400), (500, -1), (300, 50)]:
        both(gpu_lib, ctx, pairs, dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                                       band_left=w, band_right=w, zdrop=z))


def test_scoring_near_the_guard(gpu_lib, ctx):
    """Largest spreads the 16-bit guard still accepts (and one it rejects)."""
    rng = np.random.default_rng(23)
    lst = []
    for _ in range(20):
        a = rand_seq(rng, int(rng.integers(1000, 4000)))
        q = list(a)
        for k in range(len(q)):
            if rng.random() < 0.15:
                q[k] = "ACGT"[int(rng.integers(0, 4))]
        lst.append((a, "".join(q) + rand_seq(rng, 500)))
    pairs = synth.from_list(lst)
    # DESIGN.md §6.2 guard: ref16 - (spread + drift) > -17250 with
    #   spread = alpha + D*(beta + a + max(b,n)) + 4*max, drift = 70*(2*alpha + max),
    #   ref16 = -256 - (drift + 3*alpha + 2*a + max + (alpha - beta)*(D + 2));
    # at w = 280 (D = 561) this is -17040: 210 inside the limit
    both(gpu_lib, ctx, pairs, dict(match=5, mismatch=9, ambig=9, gap_open=9, gap_extend=4,
                                   band_left=280, band_right=280, zdrop=-1), expect16=True)
    # w = 290: -17500, just outside: the 32-bit kernel runs
    both(gpu_lib, ctx, pairs, dict(match=5, mismatch=9, ambig=9, gap_open=9, gap_extend=4,
                                   band_left=290, band_right=290, zdrop=-1), expect16=False)
    both(gpu_lib, ctx, pairs, dict(match=3, mismatch=12, ambig=2, gap_open=30, gap_extend=1,
                                   band_left=200, band_right=250, zdrop=200))
    both(gpu_lib, ctx, pairs, dict(match=12, mismatch=12, ambig=12, gap_open=12, gap_extend=6,
                                   band_left=500, band_right=500, zdrop=-1), expect16=False)


@pytest.mark.parametrize("sc,D,iv", [((2, 4, 4, 2), 1001, 128), ((2, 4, 6, 1), 1001, 64),
                                     ((3, 5, 6, 2), 1001, 32), ((4, 6, 6, 3), 801, 32),
                                     ((1, 3, 8, 2), 601, 64)])
def test_recentring_intervals(gpu_lib, ctx, sc, D, iv):
    """The 32-slot front re-centres every 128, 64 or 32 iterations, the longest interval the
    16-bit guard admits for the scoring and band (the drift term grows with
    the interval); every interval is bit-exact with the oracle, with and without Z-drop."""
    a, b, go, ge = sc
    rng = np.random.default_rng(31 + D + iv)
    lst = []
    for k in range(16):
        r = rand_seq(rng, int(rng.integers(2000, 5000)))
        q = "".join(c if rng.random() > 0.12 else "ACGT"[int(rng.integers(0, 4))] for c in r)
        if k % 4 == 1:
            x = int(rng.integers(200, 1500))
            q = q[:x] + q[x + int(rng.integers(5, 120)):]
        if k % 4 == 2:  # chimeric tail
            cut = int(rng.integers(len(q) // 3, len(q)))
            q = q[:cut] + rand_seq(rng, len(q) - cut)
        lst.append((r, q))
    pairs = synth.from_list(lst)
    bl = (D - 1) // 2
    for z in (-1, 150):
        params = dict(match=a, mismatch=b, ambig=b, gap_open=go, gap_extend=ge,
                      band_left=bl, band_right=D - 1 - bl, zdrop=z)
        both(gpu_lib, ctx, pairs, params, expect16=True)
        got = gpu_lib.align_pairs(ctx, pairs, params)
        assert ctx.stats()["rebase_iters"] == iv, ctx.stats()


def test_negative_stretches(gpu_lib, ctx):
    rng = np.random.default_rng(24)
    lst = [("N" * 3000, "N" * 2800), ("A" * 2000, "C" * 2000),
           ("ACGT" * 600, "N" * 700 + "ACGT" * 400), ("G" * 4000 + "ACGT" * 50, "C" * 4000)]
    for _ in range(10):
        lst.append((rand_seq(rng, 2500, "ACGTN"), rand_seq(rng, 2500, "ACGTN")))
    pairs = synth.from_list(lst)
    for w, z in [(500, -1), (500, 400), (64, -1)]:
        both(gpu_lib, ctx, pairs, dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                                       band_left=w, band_right=w, zdrop=z))
        both(gpu_lib, ctx, pairs, dict(match=1, mismatch=4, ambig=1, gap_open=6, gap_extend=2,
                                       band_left=w, band_right=w, zdrop=z))


def test_very_unequal_lengths(gpu_lib, ctx):
    rng = np.random.default_rng(25)
    lst = []
    for _ in range(16):
        a = rand_seq(rng, int(rng.integers(3000, 6000)))
        lst.append((a, a[: int(rng.integers(20, 400))]))
        lst.append((a[: int(rng.integers(20, 400))], a))
    pairs = synth.from_list(lst)
    for bl, br in [(500, 500), (511, 100), (100, 511), (0, 511)]:
        both(gpu_lib, ctx, pairs, dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                                       band_left=bl, band_right=br, zdrop=400))


def test_narrow_bands_long_pairs(gpu_lib, ctx):
    """Bands of 0-2 diagonals over long, near-identical pairs: scores climb by up to
    (a + 2 alpha)/2 per anti-diagonal for thousands of anti-diagonals, so the base
    re-centring must keep up (with bl = br = 0 every other anti-diagonal is empty and the
    32-bit kernel runs)."""
    rng = np.random.default_rng(26)
    lst = []
    for _ in range(6):
        a = rand_seq(rng, int(rng.integers(6000, 9000)))
        q = list(a)
        for k in range(0, len(q), 997):
            q[k] = "ACGT"[int(rng.integers(0, 4))]
        lst.append((a, "".join(q)))
    lst.append(("A" * 9000, "A" * 9000))
    pairs = synth.from_list(lst)
    for bl, br, exp16 in [(0, 0, False), (1, 0, True), (0, 1, True), (1, 1, True), (2, 2, True)]:
        both(gpu_lib, ctx, pairs, dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                                       band_left=bl, band_right=br, zdrop=-1), expect16=exp16)


def test_ultra_long_pair(gpu_lib, ctx):
    """A 300 kbp read (|H| beyond the 32-bit kernels' 2^20 bound) runs on the 16-bit
    kernel and matches the oracle; the 32-bit kernel refuses it with ERANGE."""
    rng = np.random.default_rng(31)
    L = 300_000
    a = rand_seq(rng, L)
    q = list(a)
    for k in range(0, L, 97):  # ~1% substitutions
        q[k] = "ACGT"[("ACGT".index(q[k]) + 1) % 4]
    pairs = synth.from_list([(a + rand_seq(rng, 200), "".join(q)), (rand_seq(rng, 5000), rand_seq(rng, 4000))])
    params = dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2, band_left=60, band_right=60, zdrop=400)
    got = gpu_lib.align_pairs(ctx, pairs, params)
    assert ctx.stats()["packed16"] == 1
    rc, exp, _ = oracle.align_batch(pairs, params)
    assert rc == 0 and got.tobytes() == exp.tobytes(), (got, exp)
    assert got[0]["score"] > (1 << 20) // 2 and got[0]["score"] > 2 * L * 0.9 - 6 * L // 97
    with pytest.raises(gpu_lib.AgathaError) as ei:
        gpu_lib.align_pairs(ctx, pairs, params, flags=gpu_lib.FORCE_32BIT)
    assert ei.value.code == gpu_lib.ERANGE

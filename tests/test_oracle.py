"""Pins for the CPU oracle (oracle/).  CPU only.

Each test pins the oracle to something other than itself (SURVEY.md §4, §8(c) "What
pins each part"):

* golden cases: brute-force path enumeration, each equal to the cited source's value;
* random tiny cases: the oracle == brute-force path enumeration (oracle/bruteforce.py),
  all five result fields, with random bands, penalties, N and Z;
* Z off + full band: the oracle == an independent row-major full DP written here from
  the plain definition (max over the table, first cell in (c, then i) order);
* closed forms: the un-terminated cell count;
* invariants: Z never raises the score, equal score => equal position, Z
  monotonicity, band nesting, R=Q with Z=0 never terminates, determinism, the
  per-anti-diagonal trace re-scanned reproduces c_term (SPEC.md S:279 analogue).
"""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import bruteforce

HERE = os.path.dirname(os.path.abspath(__file__))


def load_golden():
    rows = []
    with open(os.path.join(HERE, "golden", "cases.tsv")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            t = line.rstrip("\n").split("\t")
            R, Q = t[0], t[1]
            match, mismatch, ambig, go, ge, bl, br, z = map(int, t[2:10])
            exp = tuple(int(v) for v in t[10].split(","))
            rows.append((R, Q, dict(match=match, mismatch=mismatch, ambig=ambig, gap_open=go,
                                    gap_extend=ge, band_left=bl, band_right=br, zdrop=z), exp, t[11]))
    return rows


GOLDEN = load_golden()


@pytest.mark.parametrize("R,Q,params,expected,cite", GOLDEN, ids=[g[4][:40] for g in GOLDEN])
def test_golden(R, Q, params, expected, cite):
    rc, got = oracle.align_one(R, Q, params)
    assert rc == 0
    assert tuple(got) == expected, cite


def test_golden_file_has_paper_and_spec_rows():
    cites = " ".join(g[4] for g in GOLDEN)
    for tag in ("S:155", "S:156", "S:157", "S:158", "S:168"):
        assert tag in cites


def _rand_params(rng):
    beta = int(rng.integers(0, 4))
    alpha = int(rng.integers(beta, 8))
    return dict(match=int(rng.integers(1, 4)), mismatch=int(rng.integers(1, 6)),
                ambig=int(rng.integers(0, 6)), gap_open=alpha, gap_extend=beta,
                band_left=int(rng.integers(-1, 7)), band_right=int(rng.integers(-1, 7)),
                zdrop=int(rng.integers(-1, 8)))


def test_bruteforce_random_tiny():
    rng = np.random.default_rng(12345)
    n_checked = 0
    for _ in range(400):
        m, n = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        R = "".join(rng.choice(list("ACGTN"), m, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
        Q = "".join(rng.choice(list("ACGTN"), n, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
        if rng.random() < 0.5:
            Q = R[: n] if len(R) >= 1 else Q  # related pairs exercise long matches
        p = _rand_params(rng)
        rc, got = oracle.align_one(R, Q, p)
        assert rc == 0
        exp = bruteforce.align(R, Q, **p)
        assert tuple(got) == tuple(exp), (R, Q, p)
        n_checked += 1
    assert n_checked == 400


def test_bruteforce_zdrop_heavy():
    """Cases built to terminate: a matching prefix then garbage, Z small."""
    rng = np.random.default_rng(7)
    fired = 0
    for _ in range(150):
        k = int(rng.integers(2, 6))
        pre = "".join(rng.choice(list("ACGT"), k))
        R = pre + "".join(rng.choice(list("ACGT"), int(rng.integers(1, 5))))
        Q = pre + "".join(rng.choice(list("ACGT"), int(rng.integers(1, 5))))
        p = dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                 band_left=int(rng.integers(0, 4)), band_right=int(rng.integers(0, 4)),
                 zdrop=int(rng.integers(0, 5)))
        rc, got = oracle.align_one(R, Q, p)
        assert tuple(got) == tuple(bruteforce.align(R, Q, **p)), (R, Q, p)
        fired += got[3] >= 0
    assert fired > 20  # the sample really exercises Eq. 4


def rowmajor_fulldp(R, Q, match, mismatch, ambig, gap_open, gap_extend):
    """Plain definition with Z off and no band: H over the whole table (row-major), then
    the maximum over interior cells, first in (anti-diagonal c, then i) order."""
    m, n = len(R), len(Q)
    NEG = -(1 << 40)
    H = [[NEG] * (n + 1) for _ in range(m + 1)]
    E = [[NEG] * (n + 1) for _ in range(m + 1)]
    F = [[NEG] * (n + 1) for _ in range(m + 1)]
    H[0][0] = 0
    for i in range(1, m + 1):
        H[i][0] = -(gap_open + (i - 1) * gap_extend)
    for j in range(1, n + 1):
        H[0][j] = -(gap_open + (j - 1) * gap_extend)
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            E[i][j] = max(H[i - 1][j] - gap_open, E[i - 1][j] - gap_extend)
            F[i][j] = max(H[i][j - 1] - gap_open, F[i][j - 1] - gap_extend)
            r, q = R[i - 1], Q[j - 1]
            s = -ambig if (r == "N" or q == "N") else (match if r == q else -mismatch)
            H[i][j] = max(E[i][j], F[i][j], H[i - 1][j - 1] + s)
    best = None
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            key = (-H[i][j], i + j, i)
            if best is None or key < best[0]:
                best = (key, H[i][j], i, j)
    return best[1], best[2], best[3]


def test_full_band_equals_rowmajor_fulldp():
    rng = np.random.default_rng(99)
    batch = synth.random_short_pairs(rng, 120, 60)
    for k in range(batch.n_pairs):
        R, Q = (s.decode() for s in batch.pair(k))
        p = dict(match=2, mismatch=4, ambig=3, gap_open=5, gap_extend=1,
                 band_left=-1, band_right=-1, zdrop=-1)
        rc, got = oracle.align_one(R, Q, p)
        exp = rowmajor_fulldp(R, Q, 2, 4, 3, 5, 1)
        assert got[:3] == exp, (R, Q)
        assert got[3] == -1 and got[4] == len(R) * len(Q)
        # a band at least as wide as the sequences equals the unbanded result
        pw = dict(p, band_left=len(Q), band_right=len(R))
        assert oracle.align_one(R, Q, pw)[1] == got


def closed_form_cells(m, n, bl, br):
    # SURVEY.md [A.3]: sum_i max(0, min(n, i+bl) - max(1, i-br) + 1)
    return sum(max(0, min(n, i + bl) - max(1, i - br) + 1) for i in range(1, m + 1))


def test_cells_closed_form():
    rng = np.random.default_rng(3)
    for _ in range(200):
        m, n = int(rng.integers(1, 80)), int(rng.integers(1, 80))
        bl, br = int(rng.integers(0, 40)), int(rng.integers(0, 40))
        R = "".join(rng.choice(list("ACGT"), m))
        Q = "".join(rng.choice(list("ACGT"), n))
        rc, got = oracle.align_one(R, Q, dict(band_left=bl, band_right=br, zdrop=-1))
        assert got[4] == closed_form_cells(m, n, bl, br) == oracle.nominal_cells(m, n, bl, br)
    # symmetric m = n = L > w: L(2w+1) - w(w+1)  (SURVEY.md [A.3])
    assert oracle.nominal_cells(1000, 1000, 100, 100) == 1000 * 201 - 100 * 101 == 190_900
    assert oracle.nominal_cells(15000, 15000, 500, 500) == 14_764_500


def test_invariants_on_synthetic_pairs():
    cfg = synth.CONFIGS["C1"]
    pairs = synth.generate(cfg, 0, 40)
    base = dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2, band_left=100,
                band_right=100)
    rc, off, _ = oracle.align_batch(pairs, dict(base, zdrop=-1))
    assert rc == 0
    assert np.all(off["zdrop_antidiag"] == -1)
    prev = None
    for Z in (400, 100, 50, 10, 0):
        rc, on, _ = oracle.align_batch(pairs, dict(base, zdrop=Z))
        assert rc == 0
        assert np.all(on["score"] <= off["score"])  # Z-drop never raises the score
        same = on["score"] == off["score"]
        assert np.all(on["ref_end"][same] == off["ref_end"][same])
        assert np.all(on["query_end"][same] == off["query_end"][same])
        assert np.all(on["cells"] <= off["cells"])
        if prev is not None:  # monotone in Z: smaller Z stops no later
            t_prev = np.where(prev["zdrop_antidiag"] < 0, 1 << 30, prev["zdrop_antidiag"])
            t_now = np.where(on["zdrop_antidiag"] < 0, 1 << 30, on["zdrop_antidiag"])
            assert np.all(t_now <= t_prev)
        prev = on
    # band nesting with Z off never lowers the score
    rc, narrow, _ = oracle.align_batch(pairs, dict(base, band_left=20, band_right=20, zdrop=-1))
    assert np.all(narrow["score"] <= off["score"])
    # determinism
    rc, again, _ = oracle.align_batch(pairs, dict(base, zdrop=100), threads=3)
    rc, once, _ = oracle.align_batch(pairs, dict(base, zdrop=100), threads=1)
    assert again.tobytes() == once.tobytes()


def test_identical_sequences_never_terminate_with_z0():
    rng = np.random.default_rng(5)
    for L in (1, 2, 7, 50, 300):
        R = "".join(rng.choice(list("ACGT"), L))
        rc, got = oracle.align_one(R, R, dict(band_left=3, band_right=3, zdrop=0))
        assert got == (2 * L, L, L, -1, closed_form_cells(L, L, 3, 3))


def test_trace_rescan_reproduces_termination():
    """Re-scan the per-anti-diagonal local maxima with Eq. 4/6 written independently."""
    pairs = synth.generate(synth.CONFIGS["C1"], 40, 60)
    p = dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2, band_left=100,
             band_right=100, zdrop=100)
    n_term = 0
    for k in range(pairs.n_pairs):
        R, Q = pairs.pair(k)
        rc, got, (ts, ti) = oracle.align_one(R, Q, p, trace=True)
        m, n = len(R), len(Q)
        G = None
        term = -1
        for c in range(2, m + n + 1):
            if ti[c] < 0:
                continue
            h, i = int(ts[c]), int(ti[c])
            j = c - i
            if G and c < m + n and G[1] < i and G[2] < j and G[0] - h > 100 + 2 * abs((i - G[1]) - (j - G[2])):
                term = c
                break
            if G is None or h > G[0]:
                G = (h, i, j)
        assert (G[0], G[1], G[2], term) == got[:4]
        n_term += term >= 0
    assert n_term >= 1


def test_pack4_plain_definition():
    rc, w = oracle.pack4("ACGTACGT")
    assert rc == 0 and w.tolist() == [0x32103210]   # SPEC.md S:69 (stated value)
    rc, w = oracle.pack4("A")
    assert rc == 0 and w.tolist() == [0]
    rc, w = oracle.pack4("ACGTX")
    assert rc == oracle.ECHAR
    rc, w = oracle.pack4("ACGTX", n_map=True)
    assert rc == 0 and w.tolist() == [0x43210]
    rc, w = oracle.pack4("acgtn")
    assert w.tolist() == [0x43210]
    rc, w = oracle.pack4("AACGTN", reverse=True)      # reversed: N T G C A A
    assert w.tolist() == [0x001234]
    rng = np.random.default_rng(1)
    for _ in range(200):  # round trip
        s = "".join(rng.choice(list("ACGTN"), int(rng.integers(1, 100))))
        rc, w = oracle.pack4(s)
        dec = "".join("ACGTN"[(int(w[k // 8]) >> (4 * (k % 8))) & 15] for k in range(len(s)))
        assert dec == s
        # unused trailing nibbles are zero
        if len(s) % 8:
            assert int(w[-1]) >> (4 * (len(s) % 8)) == 0


def test_validation_errors():
    assert oracle.validate(dict(match=0)) == oracle.EINVAL
    assert oracle.validate(dict(mismatch=0)) == oracle.EINVAL
    assert oracle.validate(dict(ambig=-1)) == oracle.EINVAL
    assert oracle.validate(dict(gap_open=1, gap_extend=2)) == oracle.EINVAL
    assert oracle.validate(dict(gap_extend=-1, gap_open=0)) == oracle.EINVAL
    assert oracle.validate(dict()) == oracle.OK
    assert oracle.align_one("", "A", {})[0] == oracle.EEMPTY
    assert oracle.align_one("ACGT", "AXGT", {})[0] == oracle.ECHAR
    assert oracle.align_batch(synth.from_list([]), {})[0] == oracle.EEMPTY


def load_variants():
    rows = []
    with open(os.path.join(HERE, "golden", "variants.tsv")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            t = line.rstrip("\n").split("\t")
            bl, br, z, var = map(int, t[2:6])
            rows.append((t[0], t[1], dict(band_left=bl, band_right=br, zdrop=z, variant=var),
                         tuple(int(v) for v in t[6].split(",")), t[7]))
    return rows


VARIANTS = load_variants()


@pytest.mark.parametrize("R,Q,params,expected,cite", VARIANTS, ids=[v[4][:40] for v in VARIANTS])
def test_variant_golden(R, Q, params, expected, cite):
    """The minimap2-like alternatives (NEXT #4) on SURVEY B.2's discriminators."""
    rc, got = oracle.align_one(R, Q, params)
    assert rc == 0 and tuple(got) == expected, cite


def test_variants_vs_bruteforce_random():
    rng = np.random.default_rng(4321)
    for _ in range(300):
        m, n = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        R = "".join(rng.choice(list("ACGTN"), m, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
        Q = "".join(rng.choice(list("ACGTN"), n, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
        p = _rand_params(rng)
        p["variant"] = int(rng.integers(0, 8))
        rc, got = oracle.align_one(R, Q, p)
        assert tuple(got) == tuple(bruteforce.align(R, Q, **p)), (R, Q, p)


# oracle_align_batch (the batch driver every GPU parity test checks against) is pinned
# row by row: it slices pairs by the offsets, reorders them longest first over its worker
# threads and scatters each record back to out[k].  A slicing, ordering or scatter
# mistake would put some pair's record in another pair's row, so every row must equal
# both the single-pair oracle and the brute-force path enumeration of THAT pair.
def test_align_batch_rows_equal_align_one_and_bruteforce():
    rng = np.random.default_rng(2024)
    for trial in range(6):
        pairs_l = []
        for _ in range(70):
            m, n = int(rng.integers(1, 7)), int(rng.integers(1, 7))
            R = "".join(rng.choice(list("ACGTN"), m, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
            Q = "".join(rng.choice(list("ACGTN"), n, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
            if rng.random() < 0.4:
                Q = R[:n]
            pairs_l.append((R, Q))
        # unequal lengths in shuffled order: the longest-first reorder permutes the rows
        lens = [len(r) + len(q) for r, q in pairs_l]
        assert sorted(lens, reverse=True) != lens
        p = _rand_params(rng)
        batch = synth.from_list(pairs_l)
        for threads in (1, 3, 8):
            rc, res, status = oracle.align_batch(batch, p, threads=threads)
            assert rc == 0 and not status.any()
            for k, (R, Q) in enumerate(pairs_l):
                rc1, one = oracle.align_one(R, Q, p)
                assert rc1 == 0
                assert tuple(res[k].tolist()) == tuple(one), (trial, threads, k)
                if threads == 1:
                    assert tuple(res[k].tolist()) == tuple(bruteforce.align(R, Q, **p)), (trial, k)


def test_align_batch_rows_equal_align_one_on_c1_slice():
    cfg = synth.CONFIGS["C1"]
    pairs = synth.generate(cfg, 0, 48)
    params = vars(cfg.scoring)
    rc, res, _ = oracle.align_batch(pairs, params, threads=4)
    assert rc == 0
    assert len(set(res["cells"].tolist())) > 40  # rows are distinguishable
    for k in range(pairs.n_pairs):
        R, Q = pairs.pair(k)
        assert tuple(res[k].tolist()) == tuple(oracle.align_one(R, Q, params)[1]), k


# NEXT #4: minimap2-style end scores (reading R19), pinned by brute force path
# enumeration on random tiny pairs, by hand-derived golden rows and by a closed form.
def load_ends():
    rows = []
    with open(os.path.join(os.path.dirname(__file__), "golden", "ends.tsv")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            R, Q, bl, br, z, exp, cite = line.rstrip("\n").split("\t")
            rows.append((R, Q, dict(match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                                    band_left=int(bl), band_right=int(br), zdrop=int(z)),
                         tuple(int(x) for x in exp.split(",")), cite))
    return rows


ENDS_GOLDEN = load_ends()


@pytest.mark.parametrize("R,Q,params,expected,cite", ENDS_GOLDEN)
def test_ends_golden(R, Q, params, expected, cite):
    rc, _, ends = oracle.align_one_ends(R, Q, params)
    assert rc == 0
    assert tuple(ends) == expected, cite


def test_ends_vs_bruteforce_random_tiny():
    rng = np.random.default_rng(777)
    n_end = 0
    for _ in range(400):
        m, n = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        R = "".join(rng.choice(list("ACGTN"), m, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
        Q = "".join(rng.choice(list("ACGTN"), n, p=[0.24, 0.24, 0.24, 0.24, 0.04]))
        if rng.random() < 0.5:
            Q = R[:n]
        p = _rand_params(rng)
        rc, res, ends = oracle.align_one_ends(R, Q, p)
        assert rc == 0
        exp_res, exp_ends = bruteforce.align_ends(R, Q, **p)
        assert tuple(res) == tuple(exp_res) and tuple(ends) == tuple(exp_ends), (R, Q, p)
        n_end += ends[4] != oracle.NO_SCORE
    assert n_end > 100  # the sample reaches (m, n) often


def test_ends_closed_form_identical_and_batch_rows():
    """R = Q, full band, Z off: every end score is a*n at (n, n); batch rows equal single rows."""
    rng = np.random.default_rng(3)
    lst = []
    for L in (1, 2, 7, 33, 150):
        s = "".join(rng.choice(list("ACGT"), L))
        lst.append((s, s))
        rc, res, ends = oracle.align_one_ends(s, s, dict(match=3, band_left=-1, band_right=-1))
        assert ends == (3 * L, L, 3 * L, L, 3 * L)
    lst += [("ACGTTACG", "ACGTACG"), ("A" * 30, "A" * 5), ("GATTACA" * 9, "GATACA" * 9)]
    pairs = synth.from_list(lst)
    p = dict(match=2, mismatch=4, gap_open=4, gap_extend=2, band_left=3, band_right=5, zdrop=6)
    rc, res, ends, _ = oracle.align_batch_ends(pairs, p, threads=3)
    assert rc == 0
    rc0, res0, _ = oracle.align_batch(pairs, p)
    assert res.tobytes() == res0.tobytes()  # the records do not depend on the ends output
    for k, (R, Q) in enumerate(lst):
        _, r1, e1 = oracle.align_one_ends(R, Q, p)
        assert tuple(res[k].tolist()) == tuple(r1) and tuple(ends[k].tolist())[:5] == tuple(e1), k

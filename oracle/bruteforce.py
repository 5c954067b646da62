"""Brute-force path enumeration: an oracle-independent pin for tiny inputs.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

H(i,j) is computed WITHOUT any recurrence: it is the maximum, over every move path
from (0,0) to (i,j) that visits only in-band cells of the table, of the path score,
where a diagonal move into (x,y) scores S(R[x],Q[y]) and every
maximal run of k consecutive vertical (or horizontal) moves costs
alpha + (k-1)*beta ("A gap has to be first initiated ... ('gap
open') and can be extended by adjacent insertions/deletions ('gap extend')";
Eq. 2-3 symbols alpha, beta, l.224-226).  The origin has score 0.

The result tuple is then produced by a separate scan over the anti-diagonals that
applies Eq. 4-6 with the DESIGN.md readings: interior cells
only, local argmax ties to the smallest i, strict global update, strict position
gating, no check at c = m+n, empty anti-diagonals skipped.
"""
from __future__ import annotations

from functools import lru_cache

NEG_INF = float("-inf")


def _code(ch: str) -> int:
    return "ACGTN".index(ch.upper())


def substitution(r: str, q: str, match: int, mismatch: int, ambig: int) -> int:
    cr, cq = _code(r), _code(q)
    if cr == 4 or cq == 4:
        return -ambig
    return match if cr == cq else -mismatch


def path_table(R: str, Q: str, match=2, mismatch=4, ambig=None, gap_open=4, gap_extend=2,
               band_left=-1, band_right=-1):
    """Return {(i,j): best path score} for every in-band cell of the (m+1)x(n+1) table."""
    ambig = mismatch if ambig is None else ambig
    m, n = len(R), len(Q)
    bl = band_left if band_left >= 0 else 10 ** 9
    br = band_right if band_right >= 0 else 10 ** 9

    def inband(x, y):
        return 0 <= x <= m and 0 <= y <= n and -bl <= x - y <= br

    # Enumerate move paths by depth-first search.  The only pruning is dominance: a
    # partial path that reaches the same cell with the same last-move kind and a score
    # no higher than one already explored has no extension that scores higher (the
    # cost of every later move depends only on the cell and the last-move kind).
    best = {}
    seen = {}

    def dfs(x, y, score, last, run):
        st = (x, y, last)
        if st in seen and seen[st] >= score:
            return
        seen[st] = score
        key = (x, y)
        if key not in best or score > best[key]:
            best[key] = score
        # diagonal move
        if inband(x + 1, y + 1):
            dfs(x + 1, y + 1, score + substitution(R[x], Q[y], match, mismatch, ambig), "D", 0)
        # vertical move (consumes R)
        if inband(x + 1, y):
            cost = gap_extend if last == "V" else gap_open
            dfs(x + 1, y, score - cost, "V", run + 1 if last == "V" else 1)
        # horizontal move (consumes Q)
        if inband(x, y + 1):
            cost = gap_extend if last == "H" else gap_open
            dfs(x, y + 1, score - cost, "H", run + 1 if last == "H" else 1)

    dfs(0, 0, 0, "O", 0)
    return best


def result_from_table(table, m: int, n: int, band_left=-1, band_right=-1, gap_extend=2, zdrop=-1,
                      variant=0):
    """Apply Eq. 4-6 to a table of H values (interior cells only).  ``variant`` bits select
    the minimap2-like alternatives (1: gating <=, 2: the max starts at the origin,
    4: Eq. 4 also tested at c = m+n)."""
    bl = band_left if band_left >= 0 else 10 ** 9
    br = band_right if band_right >= 0 else 10 ** 9
    G = (0, 0, 0) if variant & 2 else None  # (H, i, j)
    last = m + n + 1 if variant & 4 else m + n
    term = -1
    cells = 0
    for c in range(2, m + n + 1):
        diag = [(i, c - i) for i in range(1, m + 1)
                if 1 <= c - i <= n and -bl <= i - (c - i) <= br]
        if not diag:
            continue
        cells += len(diag)
        vals = [(table[(i, j)], i, j) for (i, j) in diag]
        best_h = max(v[0] for v in vals)
        li, lj = min((i, j) for (h, i, j) in vals if h == best_h)
        gated = (G[1] <= li and G[2] <= lj) if (G is not None and variant & 1) else \
            (G is not None and G[1] < li and G[2] < lj)
        if G is not None and zdrop >= 0 and c < last and gated:
            if G[0] - best_h > zdrop + gap_extend * abs((li - G[1]) - (lj - G[2])):
                term = c
        if G is None or best_h > G[0]:
            G = (best_h, li, lj)
        if term >= 0:
            break
    return (G[0], G[1], G[2], term, cells)


def align(R: str, Q: str, match=2, mismatch=4, ambig=None, gap_open=4, gap_extend=2,
          band_left=-1, band_right=-1, zdrop=-1, variant=0):
    """Full result tuple (score, ref_end, query_end, zdrop_antidiag, cells) by brute force."""
    table = path_table(R, Q, match, mismatch, ambig, gap_open, gap_extend, band_left, band_right)
    return result_from_table(table, len(R), len(Q), band_left, band_right, gap_extend, zdrop, variant)


NO_SCORE = -(1 << 30)


def ends_from_table(table, m: int, n: int, c_end: int):
    """NEXT #4 end scores (reading R19) from a table of H values: over the in-band
    cells with i + j <= c_end, mqe = max H(i, n) (smallest i on ties), mte = max H(m, j)
    (smallest j on ties), end_score = H(m, n); absent -> (NO_SCORE, -1)."""
    q = [(table[(i, n)], i) for i in range(1, m + 1) if (i, n) in table and i + n <= c_end]
    t = [(table[(m, j)], j) for j in range(1, n + 1) if (m, j) in table and m + j <= c_end]
    mqe, mqe_i = (NO_SCORE, -1)
    if q:
        mqe = max(v for v, _ in q)
        mqe_i = min(i for v, i in q if v == mqe)
    mte, mte_j = (NO_SCORE, -1)
    if t:
        mte = max(v for v, _ in t)
        mte_j = min(j for v, j in t if v == mte)
    end = table[(m, n)] if (m, n) in table and m + n <= c_end else NO_SCORE
    return (mqe, mqe_i, mte, mte_j, end)


def align_ends(R: str, Q: str, match=2, mismatch=4, ambig=None, gap_open=4, gap_extend=2,
               band_left=-1, band_right=-1, zdrop=-1, variant=0):
    """(result tuple, end-score tuple) by brute force."""
    table = path_table(R, Q, match, mismatch, ambig, gap_open, gap_extend, band_left, band_right)
    res = result_from_table(table, len(R), len(Q), band_left, band_right, gap_extend, zdrop, variant)
    c_end = res[3] if res[3] >= 0 else len(R) + len(Q)
    return res, ends_from_table(table, len(R), len(Q), c_end)

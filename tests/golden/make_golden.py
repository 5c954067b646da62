"""Write tests/golden/cases.tsv.  Calls only oracle/ (the brute-force path enumerator).

Each row's expected tuple (score, ref_end, query_end, zdrop_antidiag, cells) is computed
by ``oracle.bruteforce`` (path enumeration + a separate Eq. 4-6 scan), and then checked
against the value stated by the cited source before the file is written:

  * SPEC.md worked examples — SPEC.md's own stated values
    (S:156 is stated wrongly there; SURVEY.md Appendix A.1 gives the corrected value);
  * values the survey derived by a separate brute force.

Scoring is the paper's example (§2.1 l.223-226: match +2, mismatch -4,
alpha 4, beta 2) unless a row says otherwise; N penalty = mismatch.

Run:  python tests/golden/make_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.setrecursionlimit(100000)

from oracle import bruteforce  # noqa: E402

FULL = 9  # a band of 9 is "full" for these lengths

# (R, Q, band_left, band_right, zdrop, gap_open, ambig, stated, citation)
CASES = [
    ("ACGT", "ACGT", FULL, FULL, -1, 4, 4, (8, 4, 4, -1, 16), "SPEC.md S:155; SURVEY B.1"),
    ("AAAA", "AATA", FULL, FULL, -1, 4, 4, (4, 2, 2, -1, 16), "SPEC.md S:156 corrected (SURVEY A.1, B.1)"),
    ("A", "T", FULL, FULL, -1, 4, 4, (-4, 1, 1, -1, 1), "SPEC.md S:168; SURVEY B.1"),
    ("AAAA" + "C" * 12, "AAAA" + "G" * 12, 2, 2, 4, 4, 4, (8, 4, 4, 11, 23), "SPEC.md S:157; SURVEY A.1, B.1"),
    ("ACGTACGTACGTAC", "ACGTACGTACGTAC", 3, 3, 0, 4, 4, (28, 14, 14, -1, 86), "SPEC.md S:158 (Z=0, R=Q never terminates); SURVEY A.1"),
    ("ACGTACGT", "ACGTACGT", 0, 0, -1, 4, 4, (16, 8, 8, -1, 8), "SURVEY B.1: w=0, odd anti-diagonals empty"),
    ("ACGTTACG", "ACGTACG", 1, 1, -1, 4, 4, (10, 8, 7, -1, 20), "SURVEY B.1: one deletion"),
    ("ACGTTACG", "ACGTACG", 0, 2, -1, 4, 4, (10, 8, 7, -1, 20), "SURVEY B.1: br bounds i-j>0"),
    ("ACGTTACG", "ACGTACG", 2, 0, -1, 4, 4, (8, 4, 4, -1, 18), "SURVEY B.1: band on the other side"),
    ("ACNGT", "ACNGT", FULL, FULL, -1, 4, 4, (4, 2, 2, -1, 25), "SURVEY B.1/B.2 #6,#13: N==N no match; global tie -> earliest c"),
    ("NNNN", "NNNN", FULL, FULL, -1, 4, 4, (-4, 1, 1, -1, 16), "SURVEY B.1: all-N"),
    ("AAAAAAAAAA", "AAA", 1, 1, -1, 4, 4, (6, 3, 3, -1, 8), "SURVEY B.1: |m-n|>w, trailing empty anti-diagonals"),
    ("ACGTACGTAC", "ACGTA" + "A" * 11, 3, 3, 4, 4, 4, (10, 5, 5, 14, 41), "SURVEY B.1: Z-drop with indel band"),
    ("GATTACA", "GATACA", 2, 2, -1, 4, 4, (8, 7, 6, -1, 26), "SURVEY B.1: gap in the optimum"),
    ("GCTG", "CT", 2, 3, 4, 4, 4, (0, 3, 2, -1, 8), "SURVEY B.2 #4: origin excluded from the max"),
    ("CGGGTT", "GCCATA", 2, 3, 0, 4, 4, (-2, 1, 2, 5, 9), "SURVEY B.2 #5: local tie -> smallest i"),
    ("CGGACT", "CCTAG", 3, 3, 0, 4, 4, (2, 1, 1, 4, 6), "SURVEY B.2 #8: strict position gating"),
    ("TTA", "GCT", 3, 2, 4, 4, 4, (-4, 1, 1, -1, 9), "SURVEY B.2 #9: no check at c=m+n"),
    ("ACGTTACG", "ACGTACG", 1, 1, -1, 6, 4, (8, 4, 4, -1, 20), "SURVEY B.2 #1: alpha=6"),
    ("GATTACA", "GATACA", 2, 2, -1, 6, 4, (6, 3, 3, -1, 26), "SURVEY B.2 #1: alpha=6"),
    ("ACNGT", "ACNGT", FULL, FULL, -1, 4, 1, (7, 5, 5, -1, 25), "SURVEY B.2 #13: n=1"),
]


# SURVEY.md Appendix B.2 "Alternative" column: the same discriminator inputs under the
# minimap2-like readings (NEXT #4), selected by the variant bits
# 1 = non-strict gating, 2 = max starts at the origin, 4 = Eq. 4 also at c = m+n.
VARIANT_CASES = [
    ("GCTG", "CT", 2, 3, 4, 2, (0, 0, 0, 4, 5), "SURVEY B.2 #4 alternative: origin counts in the max"),
    ("CGGACT", "CCTAG", 3, 3, 0, 1, (2, 1, 1, 3, 3), "SURVEY B.2 #8 alternative: non-strict gating"),
    ("TTA", "GCT", 3, 2, 4, 4, (-4, 1, 1, 6, 9), "SURVEY B.2 #9 alternative: checked at c = m+n"),
    # the default readings on the same inputs (variant 0) for contrast
    ("GCTG", "CT", 2, 3, 4, 0, (0, 3, 2, -1, 8), "SURVEY B.2 #4 SPEC reading"),
    ("CGGACT", "CCTAG", 3, 3, 0, 0, (2, 1, 1, 4, 6), "SURVEY B.2 #8 SPEC reading"),
    ("TTA", "GCT", 3, 2, 4, 0, (-4, 1, 1, -1, 9), "SURVEY B.2 #9 SPEC reading"),
]


# NEXT #4 end scores (reading R19, minimap2's mqe / mte / end score; outside the
# paper): (R, Q, band_left, band_right, zdrop, stated (mqe, mqe_i, mte, mte_j, end), why).
# The stated values are derived by hand: R = Q gives 2n at (n, n) on both ends; a single
# cell is its own end; a pair terminated before any end cell has none; SURVEY B.1's global
# max of the one-deletion pair sits at (8, 7), the only reference-end cell in its band.
NO = -(1 << 30)
ENDS_CASES = [
    ("ACGT", "ACGT", FULL, FULL, -1, (8, 4, 8, 4, 8), "R = Q: 2n at (n, n) (SPEC.md S:155)"),
    ("A", "T", FULL, FULL, -1, (-4, 1, -4, 1, -4), "one cell: both ends and the end score (S:168)"),
    ("AAAA" + "C" * 12, "AAAA" + "G" * 12, 2, 2, 4, (NO, -1, NO, -1, NO),
     "terminated at c = 11 (S:157) before any end cell (c >= 17)"),
    ("AAAAAAAAAA", "AAA", 1, 1, -1, (6, 3, NO, -1, NO),
     "query end at i = 2..4: H(3,3) = 6 > H(4,3) = 2 > H(2,3) = 0; reference end out of band"),
    ("ACGTTACG", "ACGTACG", 1, 1, -1, (10, 8, 10, 7, 10),
     "SURVEY B.1: max 10 first reached at (8, 7), the only cell with i = m in the band"),
]


def write_ends():
    rows = []
    for R, Q, bl, br, z, stated, cite in ENDS_CASES:
        _, got = bruteforce.align_ends(R, Q, match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                                       band_left=bl, band_right=br, zdrop=z)
        if tuple(got) != tuple(stated):
            raise SystemExit(f"brute force {got} disagrees with stated {stated} for {R}/{Q} ({cite})")
        rows.append("\t".join([R, Q, str(bl), str(br), str(z), ",".join(str(x) for x in got), cite]))
    hdr = ("# R\tQ\tband_left\tband_right\tzdrop\tends(mqe,mqe_i,mte,mte_j,end_score)\tcitation  (scoring 2/4/4/4/2)\n"
           "# written by tests/golden/make_golden.py (oracle.bruteforce); each row equals its stated value\n")
    with open(os.path.join(HERE, "ends.tsv"), "w") as f:
        f.write(hdr + "\n".join(rows) + "\n")


def write_variants():
    rows = []
    for R, Q, bl, br, z, var, stated, cite in VARIANT_CASES:
        got = bruteforce.align(R, Q, match=2, mismatch=4, ambig=4, gap_open=4, gap_extend=2,
                               band_left=bl, band_right=br, zdrop=z, variant=var)
        if tuple(got) != tuple(stated):
            raise SystemExit(f"brute force {got} disagrees with stated {stated} for {R}/{Q} ({cite})")
        rows.append("\t".join([R, Q, str(bl), str(br), str(z), str(var),
                               ",".join(str(x) for x in got), cite]))
    hdr = ("# R\tQ\tband_left\tband_right\tzdrop\tvariant\texpected\tcitation  (scoring 2/4/4/4/2)\n"
           "# written by tests/golden/make_golden.py (oracle.bruteforce); each row equals SURVEY B.2\n")
    with open(os.path.join(HERE, "variants.tsv"), "w") as f:
        f.write(hdr + "\n".join(rows) + "\n")


def main():
    rows = []
    for R, Q, bl, br, z, go, amb, stated, cite in CASES:
        got = bruteforce.align(R, Q, match=2, mismatch=4, ambig=amb, gap_open=go, gap_extend=2,
                               band_left=bl, band_right=br, zdrop=z)
        if tuple(got) != tuple(stated):
            raise SystemExit(f"brute force {got} disagrees with stated {stated} for {R}/{Q} ({cite})")
        rows.append("\t".join([R, Q, "2", "4", str(amb), str(go), "2", str(bl), str(br), str(z),
                               ",".join(str(v) for v in got), cite]))
    hdr = ("# R\tQ\tmatch\tmismatch\tambig\tgap_open\tgap_extend\tband_left\tband_right\tzdrop\t"
           "expected(score,ref_end,query_end,zdrop_antidiag,cells)\tcitation\n"
           "# written by tests/golden/make_golden.py (oracle.bruteforce path enumeration);\n"
           "# every row also equals the value stated by its cited source.\n")
    with open(os.path.join(HERE, "cases.tsv"), "w") as f:
        f.write(hdr + "\n".join(rows) + "\n")
    print(f"wrote {len(rows)} cases")
    write_variants()
    write_ends()


if __name__ == "__main__":
    main()

"""Edge-case SASS listings for parity tests: a candidate at the top or the bottom of
the schedule (boundary rejections), no legal move, only candidates, a control-flow
cut, and the smallest listing.  tests/golden/make_edge_golden.py runs the reference
on them; tests/test_oracle.py and tests/test_engine_gpu.py check against that."""
EDGE_LISTINGS = {
    "two_instructions": """\
[B------:R-:W-:-:S04] IADD3 R5, R6, 0x1, RZ ;
[B------:R-:W-:-:S01] STG.E [R2.64], R7 ;
""",
    "candidate_at_top": """\
[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;
[B------:R-:W-:-:S04] IADD3 R5, R6, 0x1, RZ ;
[B------:R-:W-:-:S04] IADD3 R8, R9, 0x1, RZ ;
[B0-----:R-:W-:-:S01] IADD3 R10, R4, 0x1, RZ ;
""",
    "candidate_at_bottom": """\
[B------:R-:W-:-:S04] IADD3 R5, R6, 0x1, RZ ;
[B------:R-:W-:-:S04] IADD3 R8, R9, 0x1, RZ ;
[B------:R-:W-:-:S01] STG.E [R2.64], R7 ;
""",
    "no_legal_move": """\
[B------:R-:W-:-:S04] IADD3 R7, R6, 0x1, RZ ;
[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;
[B0-----:R-:W-:-:S04] IADD3 R7, R4, R7, RZ ;
""",
    "all_candidates": """\
[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;
[B------:R-:W1:-:S01] LDG.E R5, [R2.64+0x4] ;
[B------:R-:W2:-:S01] LDG.E R6, [R2.64+0x8] ;
[B------:R-:W3:-:S01] LDG.E R7, [R2.64+0xc] ;
""",
    "cut_by_branch": """\
[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;
[B------:R-:W-:-:S04] IADD3 R5, R6, 0x1, RZ ;
[B------:R-:W-:-:S05] BRA `(.L_x_0) ;
.L_x_0:
[B------:R-:W-:-:S04] IADD3 R8, R9, 0x1, RZ ;
[B------:R-:W1:-:S01] LDG.E R11, [R2.64+0x10] ;
[B------:R-:W-:-:S04] IADD3 R12, R13, 0x1, RZ ;
[B01----:R-:W-:-:S01] IADD3 R14, R4, R11, RZ ;
""",
}

"""CPU oracle for the block extractor -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
`--impl reference` arm) may import this package, and only as the checker or the
timed CPU reference.  The product package (paper_2402_14607_b200) never imports
it; see DESIGN.md section "Oracle".
"""

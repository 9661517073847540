"""CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle/tm_oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  The product
(paper_2604_12241_b200) never imports it: it is the checker, not a fallback.
"""

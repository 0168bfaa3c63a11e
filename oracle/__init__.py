"""CPU oracle of the ABFT stencil method -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package (see abft_oracle.h).
"""

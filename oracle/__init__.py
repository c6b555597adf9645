"""CPU oracle -- TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).

Never imported by the product package paper_1907_01729_b200.
"""

"""CPU oracle for the GranularGym timestep — test infrastructure only.

Importable from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg.  Never imported by the product package.
"""

"""Test infrastructure: the CPU oracle for the reduced-ring ReLU path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
See hb_oracle.py for what it restates and how its parity is pinned.
"""

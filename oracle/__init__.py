"""Test-infrastructure oracle package (see spcp_oracle.py header).

Not part of the product: only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs import it.
"""

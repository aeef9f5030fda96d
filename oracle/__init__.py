"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the HBP hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  The product package never imports it.  See oracle.py.
"""

"""CPU oracle — TEST INFRASTRUCTURE ONLY. See oracle/oracle.py and oracle/oracle.c.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""

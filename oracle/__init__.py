"""TEST INFRASTRUCTURE: CPU parity checkers (C restatement + compiled reference).

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""

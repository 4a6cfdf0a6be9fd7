"""CPU oracle for the parity tests (TEST INFRASTRUCTURE -- never imported by the product).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this package.  See oracle/winofuse_oracle.c for the file:line map
onto the reference.
"""

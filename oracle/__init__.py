"""CPU oracle for the PA hash path -- TEST INFRASTRUCTURE ONLY.

`modpa_ssa.c` restates the reference's algorithm (SSA over Z/(2^N'+1),
pkg/src/modpa/ntt.py; dispatch and primitives pkg/src/modpa/bignum.py;
compress pkg/src/modpa/pa.py:175-190) in plain C.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this package; the
product path never does.  Pinned against reference-generated golden vectors
in tests/test_oracle.py.
"""
from .oracle import available, build, compress, compress_batch, mul, plan  # noqa: F401

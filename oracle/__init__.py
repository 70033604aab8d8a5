"""CPU oracle for APML / CUDA-APML (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl
reference`` legs may import this package.  The product path
(``paper_2512_19743_b200``) never imports it.  See oracle/apml_oracle.c for the
algorithm and its PAPER.md citations.
"""
from .oracle import (  # noqa: F401
    OracleConfig, SparsePlan, build_oracle, dense_forward, sparse_forward, batch, temperature, line,
)

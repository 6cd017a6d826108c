"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain CPU Pbit (arXiv cs/0511020) used to prove the CUDA path right.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_cs_0511020_b200`` never imports it and shares no code with it.

See ``oracle/pbit_oracle.c`` for the paper-literal algorithm and its citations.
"""
from .oracle import (  # noqa: F401
    ORACLE_NULL,
    OracleError,
    bits,
    build,
    list_order,
    memory_bound_T,
    pbit_sort,
    pbit_sort_par,
    repair_back,
    split_once,
    validate_list,
)

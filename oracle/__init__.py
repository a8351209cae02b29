"""TEST INFRASTRUCTURE ONLY: CPU oracles for the SCC hot path.

Two oracles live here, both double precision:

* ``port``      -- ``oracle/scc_oracle.c``, a plain-C restatement of the
                   reference (proj/core/src/kernel.cpp, config.cpp, cycle.cpp),
                   built into ``oracle/_build/libscc_oracle.so``.
* ``reference`` -- the reference library itself, compiled from the untouched
                   sources under /root/reference by ``oracle/Makefile`` into
                   ``oracle/_ref/libsccl_ref.so`` and reached through
                   ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this package.  The product package
``paper_2101_00745_b200`` never does.
"""
from .oracle import (  # noqa: F401
    OracleConfig,
    OracleError,
    PortOracle,
    RefOracle,
    build,
    load_port,
    load_ref,
)

"""CPU oracle for the butterfly-factorization hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain NumPy, the reference algorithm of
arxiv/paper_1502_01379 (package ``butterfly`` under /root/reference/pkg/src)
for the path this repository accelerates:

* ``oracle.partition`` — dyadic geometry (reference ``partition.py``) and the
  level geometry table (reference ``construct.py:216-227``);
* ``oracle.chain``     — the factor-apply chain and its adjoint (reference
  ``factors.py:49-237``);
* ``oracle.entries``   — entry oracles K(x, xi) = exp(2 pi i Phi) for the
  BASELINE.json configs (reference ``kernels.py:23-42`` plus the config-1 DFT
  convention the reference lacks);
* ``oracle.lowrank``   — pivot selection, bases, floored pseudo-inverse,
  randomized sampling SVD (reference ``lowrank.py:79-293``);
* ``oracle.construct`` — middle-level sampling and the recursive block SVDs
  (reference ``construct.py:26-259``).

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
fixtures in ``tests/golden/`` produced by running the reference itself
(``oracle/gen_golden.py``, committed), plus the reference's own known-answer
tests (``pkg/tests/test_kernels.py:13-17``, ``test_factors.py:16-89``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package — and only as the checker or
the timed CPU reference arm. The product package ``paper_1502_01379_b200`` never
imports it: its compute path is the CUDA library behind ``include/bfly.h``.
"""

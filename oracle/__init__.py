"""CPU oracle for the restructured-BN training path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_1807_01702_b200``) never imports it and fails loudly when its CUDA
library is missing.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
(``/root/reference/pkg/src/bnfuse``, numpy) in the build container and writes
fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
restatement against them.
"""

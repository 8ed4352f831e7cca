"""CPU oracle for the batched strategy evaluator — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package, and only as the checker / CPU baseline. The product
package (paper_2509_00217_b200) never imports it; it fails loudly when its
CUDA library is missing instead of falling back here.

Pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""

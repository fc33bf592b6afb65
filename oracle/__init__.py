"""CPU oracle for the streaming-SVD hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithm of the reference
`parsvd` package (arXiv 2108.08845 / PyParSVD, `/root/reference/pkg/src/parsvd`)
for the path BASELINE.json's north star names: the serial and row-parallel
streaming SVD update (deterministic and the randomized composition R9).
Each function cites the reference file:line it follows.

Pinning: the restatement is checked against golden vectors produced by the
live reference (tests/golden/make_golden.py imports /root/reference in the
build container; the .npz fixtures travel, the reference does not) — see
tests/test_oracle_golden.py.

Only tests/, __graft_entry__.smoke() and bench.py's `cpu_baseline` /
`--impl reference` leg may import this package, and only as the checker /
CPU baseline.  The product package (paper_2108_08845_b200) never imports it
and has no CPU fallback.
"""

from .core import (  # noqa: F401
    burgers_matrix, burgers_solution, partition_bounds, ref_omega, ref_qr,
    ref_svd, ref_low_rank_svd, ref_range, ref_stream_init, ref_stream_update,
    ref_stream_all, ref_rand_stream_init, ref_rand_stream_update,
    ref_rand_stream_all, ref_parallel_stream_all, sigma_rel_err,
    sine_angles, mode_angles, aligned_mode_difference,
    ref_generate_right_vectors, ref_apmos,
)

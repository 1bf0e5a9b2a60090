"""CPU oracle for the distributed-RNG + redistribute hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything in
this package, and only as the checker (or the timed CPU baseline).  The product
package `paper_2509_07003_b200` never imports it and has no CPU fallback.

Contents
--------
* `rng_oracle`   -- NumPy restatement of `spmdsim.rng` + the index algebra of
                    `spmdsim.placement` (reference: /root/reference/pkg/src/
                    spmdsim/rng.py, placement.py).  Pure function of its inputs.
* `redist_oracle`-- NumPy restatement of the per-fiber redistribute transitions
                    (`spmdsim.dtensor._transition`, `_assemble_shards`,
                    `_local_slice`, `comm.reduce_scatter` ascending-rank sums).
* `c/`           -- plain-C restatement of Philox4x32-10 and the integer/exact
                    fills (uniform01-f32, bernoulli/dropout), built by
                    `oracle/Makefile` into `oracle/_build/liboracle_c.so`.

Pinning
-------
The restatement is pinned against (1) the Random123 known-answer vectors and the
reference's own GOLDEN_ZERO block (pkg/tests/test_rng.py:24-30), and (2) golden
fixtures produced by importing the real reference in the build container
(`tests/golden/make_golden.py`, committed together with its `.npz` outputs).
`tests/test_oracle.py` checks every fixture bit for bit.

`Normal` values depend on NumPy's float64 `log1p`/`cos` (the reference's own
dependency, unpinned `numpy>=1.24`, pkg/pyproject.toml:10-12).  The oracle calls
the same NumPy functions, so oracle and reference agree on any host; the golden
normal fixtures are only comparable on hosts whose NumPy SIMD dispatch gives the
same `log1p` bits (checked at test time, see tests/test_oracle.py).
"""

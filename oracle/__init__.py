"""CPU oracle for the fusion + property-query path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference` legs may
import this package, and only as the checker or the timed CPU reference — never as the thing
measured or shipped. The product path (`paper_2511_03126_b200`) never imports it and fails loudly
without its CUDA library.

`oracle.propfield_oracle` restates the reference algorithm (propfield, /root/reference/pkg) in
numpy + numba, function by function, citing the reference file:line each one follows. It is pinned
against the reference itself: `tests/golden/make_golden.py` imports the reference from
/root/reference in the build container and writes golden vectors; `tests/test_oracle.py` checks
the restatement against them (and directly against the reference when it is importable).

Parity status: visibility, aggregation, normalisation, similarity, softmax, regression and the
integrate_mass partials are PINNED to reference outputs. The voxel-grid mass has
no reference implementation: it is a restatement of the BASELINE definition whose parity is
UNPINNED (its indexing is pinned to the convention of sampling.py:110-123 only).
"""

"""oracle — plain, slow, obviously-correct CPU model of the compressed gradient sync.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call, link or
execute anything under ``oracle/``; the only permitted users are ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs.  The oracle shares no code, headers, tables or constants with the CUDA path in
``paper_2205_09470_b200/csrc`` and neither imports the other.  The only module both
sides use is ``gradgen`` (seeded input generation, no method arithmetic).

Every function follows a passage of PAPER.md / SPEC.md (cited as ``PAPER.md:L`` /
``SPEC.md:L``) or, where the reference is silent, a reading listed in DESIGN.md
("Readings", R-numbers == SURVEY.md §8(c) C-numbers).  All floating-point work is
IEEE-754 binary32 with round-to-nearest-even, one rounding per operation, done with
explicit ``np.float32`` operands so NumPy never widens or fuses an operation.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to something other
than itself: Table 5's ratio column, SPEC.md's worked examples, closed-form error bounds,
the residual identity p == D(C(p)) + r_new, EF telescoping, brute-force top-k over all
subsets of tiny vectors, and textbook special cases of the average.  Nothing here is
"parity unpinned" except throughput, which the paper never prints for this path.
"""
from .codec import *  # noqa: F401,F403
from .codec import __all__  # noqa: F401
from .svd import *  # noqa: F401,F403  (FP16(SVD(rho)) low-rank compressor, NEXT-1)

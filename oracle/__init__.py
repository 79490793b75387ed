"""CPU oracle for the Theano-MPI parameter exchange (arXiv 1605.08325).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_1605_08325_b200``,
``libtm.so``) may import, call, link or execute anything under ``oracle/``.  The
only permitted users are ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.

The oracle is deliberately plain and slow: pure numpy, fp32 only where the method
computes in fp32 (every fp32 step is ONE numpy float32 ufunc, i.e. one correctly
rounded IEEE operation; no fused multiply-add, no reassociation), fp16 rounding by
an integer-only bit emulation.  It follows the paper's steps in the paper's
order: partition into sub-arrays, Alltoall, sum on the owner, Allgather
(Sec. 3.2, Fig. 2 caption L252-256), with the half-precision
transfer of L262-269.  It shares no code with the CUDA path.

Modules
  fp16      -- rn16 (IEEE binary16 round-to-nearest-even) and widen (exact)
  exchange  -- partition / alltoall / allgather / ASA / ASA16 / AR averaging
  easgd     -- elastic-averaging update and arrival-order sequences
  bsp       -- momentum-SGD step followed by the exchange (one BSP iteration)
  loader    -- Alg. 1 preprocessing (mean, crop, mirror) and delivery sequence

Parity status of every function is listed in each module's header and in
DESIGN.md section "Oracle and pins".
"""

from . import fp16, exchange, easgd, bsp, loader  # noqa: F401

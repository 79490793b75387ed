"""k simulated BSP workers exchanging (averaging) their flat fp32 parameter vectors.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper anchors:
  L66-70  (Sec. 1)   data parallelism: copies of one model average their parameters
                     every iteration.
  L195-212 (Sec. 3.1) BSP: after SGD, workers synchronise and exchange parameters
                     "in a collective way".
  L227-228 (Sec. 3.2) "Synchronous parameter exchange is an array reduction problem".
  L233-237           AR: MPI Allreduce().
  L237-246, Fig. 2 caption L252-256
                     ASA: Alltoall, GPU summation of the sub-arrays (same-coloured
                     boxes), Allgather of the results.
  L262-269           ASA16: transfer at half precision, sum at full precision.
  L377-384 (Sec. 4)  AWAGD: weights are AVERAGED (1/k) after gradient descent.
  L384-389, L458-460 SUBGD: the parameter UPDATES are SUMMED (no 1/k); the mode of
                     the paper's convergence runs.  op="sum" below.

Readings of what the paper leaves open ("Readings"):
  Q1/R1  ASA16 quantises every contribution (own one included) and every rank,
         owner included, adopts widen(rn16(average)).
  Q2     both ASA16 phases carry fp16.
  Q3     average = fp32 sum, then ONE division by k (then, ASA16, rounding to fp16).
  Q4     the division is IEEE fl(s / k).
  Q5     sum in ascending source rank, starting from the rank-0 term (not +0.0).
  Q7     sub-arrays have length ceil(P/k); the last is zero-padded; pads are dropped.
  Q10    k = 1 is the identity for every strategy (nothing is transferred).

Each fp32 step below is ONE numpy float32 ufunc call (correctly rounded IEEE op).

Parity status: asa_average, asa16_average, ar_average (op avg and sum), partition/unpartition,
alltoall, allgather, wire_bytes_per_rank are pinned (tests/test_oracle_exchange.py:
SPEC worked examples, exact-rational brute force of every rounding step,
exact-arithmetic special cases, identity invariants, error bounds).
"""

import numpy as np

from .fp16 import rn16, widen

STRATEGIES = ("ar", "asa", "asa16")


# ---------------------------------------------------------------------------
# Sub-array layout (Fig. 2 "Sub-arrays of data items")
# ---------------------------------------------------------------------------

def sub_array_length(P, k):
    """ceil(P / k): every rank's sub-array has this length (Q7)."""
    return -(-P // k)


def partition(x, k):
    """Split flat buffer x (length P) into k equal sub-arrays of length ceil(P/k);
    the tail is zero-padded (+0)."""
    P = x.shape[0]
    L = sub_array_length(P, k)
    padded = np.zeros(k * L, dtype=x.dtype)
    padded[:P] = x
    return [padded[r * L:(r + 1) * L].copy() for r in range(k)]


def unpartition(slices, P):
    """Concatenate sub-arrays in rank order and drop the padding."""
    return np.concatenate(slices)[:P].copy()


# ---------------------------------------------------------------------------
# The two transfer collectives (no arithmetic)
# ---------------------------------------------------------------------------

def alltoall(send):
    """send[j][r] is the sub-array rank j sends to rank r.
    Returns recv with recv[r][j] = send[j][r] (rank r receives sub-array r from
    every rank j)."""
    k = len(send)
    return [[send[j][r] for j in range(k)] for r in range(k)]


def allgather(per_rank):
    """Every rank receives all k ranks' sub-arrays, in rank order."""
    k = len(per_rank)
    return [[per_rank[j] for j in range(k)] for _ in range(k)]


# ---------------------------------------------------------------------------
# Strategies
# ---------------------------------------------------------------------------

def _check(X):
    k = len(X)
    if k < 1:
        raise ValueError("need at least one worker")
    P = X[0].shape[0]
    for x in X:
        if x.dtype != np.float32 or x.ndim != 1 or x.shape[0] != P:
            raise ValueError("every worker buffer must be float32[P] of equal length")
    return k, P


def _sum_then_divide(received, k, op="avg"):
    """GPU summation step of Fig. 2 on one owner: ascending source rank, starting
    from the rank-0 term (Q5), then (op="avg", AWAGD) one IEEE division by k (Q3,
    Q4); op="sum" (SUBGD) stops after the sum."""
    s = received[0].copy()
    for j in range(1, k):
        s = np.add(s, received[j], dtype=np.float32)
    if op == "sum":
        return s
    if op != "avg":
        raise ValueError(op)
    return np.divide(s, np.float32(k), dtype=np.float32)


def asa_average(X, op="avg"):
    """ASA (fp32): Alltoall -> sum on owner -> Allgather, averaged by 1/k
    (op="sum": the sum, SUBGD).

    X: list of k float32[P] worker buffers.  Returns the list of k results
    (identical on every rank)."""
    k, P = _check(X)
    if k == 1:
        return [X[0].copy()]
    send = [partition(x, k) for x in X]          # sub-arrays, Fig. 2
    recv = alltoall(send)                         # rank r gets sub-array r of all ranks
    avg = [_sum_then_divide(recv[r], k, op) for r in range(k)]
    gathered = allgather(avg)
    return [unpartition(gathered[r], P) for r in range(k)]


def asa16_average(X, op="avg"):
    """ASA16 (reading R1): every sub-array is rounded to binary16 before the
    Alltoall (own one included), widened and summed in fp32 on the owner, divided
    by k, rounded to binary16 for the Allgather, and widened by every receiver
    (owner included)."""
    k, P = _check(X)
    if k == 1:
        return [X[0].copy()]
    send = [[rn16(s) for s in partition(x, k)] for x in X]   # fp16 on the wire
    recv = alltoall(send)
    avg16 = []
    for r in range(k):
        a = _sum_then_divide([widen(h) for h in recv[r]], k, op)   # fp32 summation
        avg16.append(rn16(a))                                   # fp16 on the wire
    gathered = allgather(avg16)
    return [widen(unpartition(gathered[r], P)) for r in range(k)]


def ar_average(X, op="avg"):
    """AR: the allreduce-average by definition, elementwise
    fl(...fl(fl(x0 + x1) + x2)... + x_{k-1}) / k, on every rank.  Its value equals
    asa_average's; a real Allreduce may sum in another order, so the GPU AR path
    is compared within the Q11 bound rather than bitwise."""
    k, P = _check(X)
    if k == 1:
        return [X[0].copy()]
    a = _sum_then_divide(X, k, op)
    return [a.copy() for _ in range(k)]


def exchange(X, strategy, op="avg"):
    """Dispatch by strategy name ('ar', 'asa', 'asa16'); op 'avg' (AWAGD) or
    'sum' (SUBGD)."""
    if strategy == "ar":
        return ar_average(X, op)
    if strategy == "asa":
        return asa_average(X, op)
    if strategy == "asa16":
        return asa16_average(X, op)
    raise ValueError(f"unknown strategy {strategy!r}")


def element_average(values, strategy, op="avg"):
    """Result of one element given its k per-rank values (1-D float32 array of
    length k, or [k, n] for n independent elements).  Same steps as the
    strategies above restricted to one index; used for sampled checks at full
    size.  For strategy 'ar' this is the rank-ordered definition."""
    v = np.asarray(values, dtype=np.float32)
    k = v.shape[0]
    if k == 1:
        return v[0].copy()
    if strategy in ("ar", "asa"):
        return _sum_then_divide([v[j] for j in range(k)], k, op)
    if strategy == "asa16":
        a = _sum_then_divide([widen(rn16(v[j])) for j in range(k)], k, op)
        return widen(rn16(a))
    raise ValueError(strategy)


# ---------------------------------------------------------------------------
# Traffic accounting: payload bytes each rank sends
# ---------------------------------------------------------------------------

def wire_bytes_per_rank(strategy, P, k):
    """Bytes one rank transmits in one exchange for the ASA family: the Alltoall
    sends k-1 sub-arrays, the Allgather sends its sum to k-1 ranks, each
    ceil(P/k) elements of 4 (ASA) or 2 (ASA16) bytes.  For AR the ring-allreduce
    volume 2(k-1)/k * 4P (rounded to whole sub-arrays) is returned."""
    if k == 1:
        return 0
    L = sub_array_length(P, k)
    if strategy == "asa":
        return 2 * (k - 1) * L * 4
    if strategy == "asa16":
        return 2 * (k - 1) * L * 2
    if strategy == "ar":
        return 2 * (k - 1) * L * 4
    raise ValueError(strategy)

"""Array-OL tilers: the index function of a repetitive task.

The reference has no tiler: its repetitive tasks use the identity
mapping "repetition point rho touches element rho of every vector port"
(/root/reference/pkg/src/gmodelc/refexec.py:488-514, codegen.py:150-168,
SPEC.md:334).  The north_star (BASELINE.json) and MARTE RSM
 define the general form frozen here:

    e(r, i) = (o + P . r + F . i) mod s_arr      (component-wise Euclidean mod)
    off(r, i) = sum_d e_d * prod_{d' > d} s_arr[d']            (int64, row-major)

with r the row-major unravel of the linear repetition index rho over the
task's ``repeat`` shape (partition.py:3-4) and i the row-major unravel of
the pattern index iota.  The identity tiler of the reference is
``Tiler.identity(n)`` over a 1-D port: o=0, P=[[1]], F=[[0]], pattern [1].

Output tilers must be injective over all (rho, iota) (single assignment);
unwritten output elements keep the executor's zero initialisation
(refexec.py:399-403).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

MAX_RANK = 4                 # rank limit of the C-ABI aol_tiler (include/aol_b200.h)
EXHAUSTIVE_LIMIT = 1 << 26   # (rho, iota) pairs checked exhaustively for injectivity


class TilerError(ValueError):
    pass


def _tuple2(m) -> tuple[tuple[int, ...], ...]:
    return tuple(tuple(int(v) for v in row) for row in m)


@dataclass(frozen=True)
class Tiler:
    """Unbound tiler: origin (a), paving (a x q), fitting (a x p) and the pattern shape (p).

    The array shape s_arr comes from the port it is attached to and the
    repetition shape from the task's ``repeat`` (see :meth:`bind`).
    """

    origin: tuple[int, ...]
    paving: tuple[tuple[int, ...], ...]
    fitting: tuple[tuple[int, ...], ...]
    pattern: tuple[int, ...]

    def __init__(self, origin, paving, fitting, pattern):
        object.__setattr__(self, "origin", tuple(int(v) for v in origin))
        object.__setattr__(self, "paving", _tuple2(paving))
        object.__setattr__(self, "fitting", _tuple2(fitting))
        object.__setattr__(self, "pattern", tuple(int(v) for v in pattern))

    @staticmethod
    def identity(rank: int = 1) -> "Tiler":
        """The reference's implicit tiler for a rank-1 port whose extent equals the repetition total."""
        eye = [[1 if i == j else 0 for j in range(rank)] for i in range(rank)]
        return Tiler([0] * rank, eye, [[0]] * rank, [1])

    def bind(self, array_shape, rep_shape) -> "BoundTiler":
        return BoundTiler(self, tuple(int(d) for d in array_shape),
                          tuple(int(d) for d in rep_shape))


_INJECTIVE_OK: set = set()


@dataclass(frozen=True)
class BoundTiler:
    tiler: Tiler
    array: tuple[int, ...]
    rep: tuple[int, ...]

    def __post_init__(self):
        t = self.tiler
        a, q, p = len(self.array), len(self.rep), len(t.pattern)
        if not (1 <= a <= MAX_RANK and 1 <= q <= MAX_RANK and 1 <= p <= MAX_RANK):
            raise TilerError(f"tiler ranks must be in 1..{MAX_RANK}: array {a}, repetition {q}, "
                             f"pattern {p}")
        if any(d < 1 for d in self.array + self.rep + t.pattern):
            raise TilerError("array, repetition and pattern dimensions must be >= 1")
        if len(t.origin) != a:
            raise TilerError(f"origin has {len(t.origin)} entries, array rank is {a}")
        if len(t.paving) != a or any(len(row) != q for row in t.paving):
            raise TilerError(f"paving must be {a}x{q} (array rank x repetition rank)")
        if len(t.fitting) != a or any(len(row) != p for row in t.fitting):
            raise TilerError(f"fitting must be {a}x{p} (array rank x pattern rank)")

    # -- sizes ---------------------------------------------------------------
    @property
    def pattern_total(self) -> int:
        return int(np.prod(self.tiler.pattern, dtype=np.int64))

    @property
    def rep_total(self) -> int:
        return int(np.prod(self.rep, dtype=np.int64))

    @property
    def array_total(self) -> int:
        return int(np.prod(self.array, dtype=np.int64))

    @cached_property
    def array_strides(self) -> tuple[int, ...]:
        s, acc = [], 1
        for d in reversed(self.array):
            s.append(acc)
            acc *= d
        return tuple(reversed(s))

    # -- analysis ------------------------------------------------------------
    def _extent_bounds(self):
        """Per array dim, min/max of o_d + P_d.r + F_d.i over the full (r, i) box (o reduced mod s)."""
        t = self.tiler
        lo, hi = [], []
        for d in range(len(self.array)):
            o = t.origin[d] % self.array[d]
            mn = mx = o
            for j, rj in enumerate(self.rep):
                v = t.paving[d][j] * (rj - 1)
                mn += min(0, v)
                mx += max(0, v)
            for k, pk in enumerate(t.pattern):
                v = t.fitting[d][k] * (pk - 1)
                mn += min(0, v)
                mx += max(0, v)
            lo.append(mn)
            hi.append(mx)
        return lo, hi

    @cached_property
    def wraps(self) -> bool:
        """True when some (r, i) needs the modulo (toroidal access)."""
        lo, hi = self._extent_bounds()
        return any(l < 0 or h >= s for l, h, s in zip(lo, hi, self.array))

    @cached_property
    def affine(self):
        """(c0, rep_coeffs, pat_coeffs) with off = c0 + rep_coeffs.r + pat_coeffs.i, or None if it wraps."""
        if self.wraps:
            return None
        t, st = self.tiler, self.array_strides
        c0 = sum((t.origin[d] % self.array[d]) * st[d] for d in range(len(self.array)))
        rc = tuple(sum(t.paving[d][j] * st[d] for d in range(len(self.array)))
                   for j in range(len(self.rep)))
        pc = tuple(sum(t.fitting[d][k] * st[d] for d in range(len(self.array)))
                   for k in range(len(t.pattern)))
        return c0, rc, pc

    # -- evaluation ----------------------------------------------------------
    def offsets(self, first: int = 0, count: int | None = None) -> np.ndarray:
        """int64 [count, pattern_total] flat offsets for rho in [first, first+count).

        Vectorised restatement used by the host (injectivity proofs); the
        test oracle has its own independent implementation.
        """
        if count is None:
            count = self.rep_total - first
        t = self.tiler
        rho = np.arange(first, first + count, dtype=np.int64)
        iota = np.arange(self.pattern_total, dtype=np.int64)
        r = np.stack(np.unravel_index(rho, self.rep), axis=0) if count else np.zeros((len(self.rep), 0), np.int64)
        i = np.stack(np.unravel_index(iota, t.pattern), axis=0)
        P = np.asarray(t.paving, dtype=np.int64)
        F = np.asarray(t.fitting, dtype=np.int64)
        o = np.asarray(t.origin, dtype=np.int64)
        base = o[:, None] + P @ r                      # a x count
        fit = F @ i                                    # a x pat
        e = base[:, :, None] + fit[:, None, :]         # a x count x pat
        s = np.asarray(self.array, dtype=np.int64)[:, None, None]
        e = np.mod(e, s)
        st = np.asarray(self.array_strides, dtype=np.int64)[:, None, None]
        return (e * st).sum(axis=0)

    def check_injective(self) -> None:
        """Raise TilerError unless every (rho, iota) maps to a distinct element (output tilers).
        A tiler that passed once is remembered (bound tilers are immutable values)."""
        if self in _INJECTIVE_OK:
            return
        self._check_injective()
        if len(_INJECTIVE_OK) < 4096:
            _INJECTIVE_OK.add(self)

    def _check_injective(self) -> None:
        n = self.rep_total * self.pattern_total
        if n > self.array_total:
            raise TilerError(f"output tiler writes {n} elements into an array of {self.array_total}")
        aff = self.affine
        if aff is not None:
            _, rc, pc = aff
            terms = sorted((abs(c), e - 1) for c, e in zip(rc + pc, self.rep + self.tiler.pattern)
                           if e > 1)
            reach, ok = 0, True
            for c, span in terms:
                if c <= reach:
                    ok = False
                    break
                reach += c * span
            if ok:
                return
        if n > EXHAUSTIVE_LIMIT:
            raise TilerError(f"cannot prove the output tiler injective ({n} writes exceed the "
                             f"exhaustive-check limit and the mixed-radix criterion fails)")
        offs = self.offsets().ravel()
        if np.unique(offs).size != offs.size:
            raise TilerError("output tiler is not injective: two (repetition, pattern) points "
                             "write the same array element")

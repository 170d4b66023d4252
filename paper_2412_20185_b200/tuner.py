"""DecDEC parameter tuner (§4.4 "Parameter Tuner"), retargeted to B200.

The paper tunes two knobs per linear-layer class (qkv, o, gu, d):
  * n_tb    -- thread blocks given to dynamic error compensation.  Here: the number of
               DEC CTAs of the fused layer kernel (decdec_set_dec_ctas), same role: too many
               take SMs from the base GEMV, too few under-drive the PCIe link;
  * k_chunk -- channels compensated per 1024 input channels.
Objective: maximise k_chunk while the total execution time of all linear layers
(base GEMV + compensation) stays within a target slowdown of the uncompensated baseline.

Algorithm, in the paper's order:
  Phase 1: for each metaparameter n_max (<= half the SMs), every class takes the
    largest n candidate <= n_max; a coarse search counts how many uniform +1 increments of
    k_chunk (all classes together) stay within the target.  If no n_max allows a step, the
    class with the smallest weight matrix is fixed at k_chunk = 0 and Phase 1 repeats.
  Phase 2: from the best n_max's uniform k_chunk, repeatedly try +1 on every
    non-frozen class, cheapest time increase first; a class whose increment would exceed the
    target is frozen.  Stops when every class is frozen.

This module is the search only (host logic, testable on CPU); the measured time table comes
from tools/tune.py on the GPU.  `time_fn(cls, n, k_chunk) -> µs per call` must be monotone
enough for a greedy search (the paper's assumption too).
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class LayerClass:
    name: str
    count: int   # calls per decode step (e.g. 32 blocks)
    d_in: int
    d_out: int


@dataclass
class TuneResult:
    target: float
    n_max: int
    n: dict = field(default_factory=dict)        # class -> DEC CTAs
    k_chunk: dict = field(default_factory=dict)  # class -> k_chunk
    base_us: float = 0.0                         # uncompensated step time (linear layers)
    us: float = 0.0                              # tuned step time
    phase1_steps: dict = field(default_factory=dict)  # n_max -> valid uniform steps

    @property
    def slowdown(self) -> float:
        return self.us / self.base_us - 1.0

    def table2(self) -> str:
        """The paper's Table 2 cell format: n_max / (k_qkv, k_o, k_gu, k_d) -> slowdown."""
        ks = ",".join(str(self.k_chunk[c]) for c in self.k_chunk)
        return f"{self.n_max}/({ks}) -> {100 * self.slowdown:.1f}%"


def n_candidates_paper(d_in: int, d_out: int, seg_cols: int = 256) -> list:
    """The paper's candidate set N = A ∪ B: A = 1..d_in/1024 (Top-K chunks),
    B = the n with distinct ceil(s/n) segments per block, s = d_out / 256."""
    A = set(range(1, max(1, d_in // 1024) + 1))
    s = max(1, d_out // seg_cols)
    B = {n for n in range(1, s + 1) if -(-s // -(-s // n)) == n}
    return sorted(A | B)


def _step_time(classes, time_fn, n, k):
    return sum(c.count * time_fn(c.name, n[c.name], k[c.name]) for c in classes)


def tune(classes, time_fn, target: float, n_max_values, n_candidates, k_max: int = 128,
         base_n: int | None = None) -> TuneResult:
    """classes: [LayerClass]; n_candidates(cls) -> sorted list of allowed n for that class;
    n_max_values: metaparameter values to try (Phase 1); base_n: n used for the k = 0
    baseline (the uncompensated kernel does not use DEC CTAs, so any value)."""
    names = [c.name for c in classes]
    n0 = {c.name: (base_n if base_n is not None else n_candidates(c)[0]) for c in classes}
    base = _step_time(classes, time_fn, n0, {c: 0 for c in names})
    budget = base * (1.0 + target)

    def n_for(n_max):
        out = {}
        for c in classes:
            cand = [v for v in n_candidates(c) if v <= n_max]
            out[c.name] = cand[-1] if cand else n_candidates(c)[0]
        return out

    fixed_zero = set()
    by_size = sorted(classes, key=lambda c: c.d_in * c.d_out)
    while True:  # Phase 1 (with the smallest-matrix fallback of P:311)
        steps = {}
        for n_max in n_max_values:
            n = n_for(n_max)
            s = 0
            while s < k_max:
                k = {c: (0 if c in fixed_zero else s + 1) for c in names}
                if _step_time(classes, time_fn, n, k) > budget:
                    break
                s += 1
            steps[n_max] = s
        best = max(n_max_values, key=lambda v: (steps[v], -v))
        if steps[best] > 0 or len(fixed_zero) == len(names):
            break
        nxt = next((c.name for c in by_size if c.name not in fixed_zero), None)
        if nxt is None:
            break
        fixed_zero.add(nxt)

    n = n_for(best)
    k = {c: (0 if c in fixed_zero else steps[best]) for c in names}
    frozen = set(fixed_zero)
    while len(frozen) < len(names):  # Phase 2
        cur = _step_time(classes, time_fn, n, k)
        order = sorted((c for c in classes if c.name not in frozen),
                       key=lambda c: c.count * (time_fn(c.name, n[c.name], k[c.name] + 1) -
                                                time_fn(c.name, n[c.name], k[c.name])))
        for c in order:
            if k[c.name] + 1 > k_max:
                frozen.add(c.name)
                continue
            trial = dict(k)
            trial[c.name] += 1
            t = _step_time(classes, time_fn, n, trial)
            if t > budget:
                frozen.add(c.name)
            else:
                k = trial
                cur = t
    res = TuneResult(target=target, n_max=best, n=n, k_chunk={c: k[c] for c in names}, base_us=base,
                     us=_step_time(classes, time_fn, n, k), phase1_steps=steps)
    return res


def interp_table(table: dict):
    """time_fn from a measured table {cls: {n: {k_chunk: us}}}, linear in k_chunk between
    measured points (and flat beyond the last one is NOT assumed: extrapolate the last slope)."""
    def f(cls, n, k):
        row = table[cls][n]
        ks = sorted(row)
        if k in row:
            return row[k]
        if k <= ks[0]:
            return row[ks[0]]
        for a, b in zip(ks, ks[1:]):
            if a <= k <= b:
                return row[a] + (row[b] - row[a]) * (k - a) / (b - a)
        a, b = ks[-2], ks[-1]
        return row[b] + (row[b] - row[a]) * (k - b) / (b - a)
    return f

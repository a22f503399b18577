"""QSpec cost model with a MEASURED B200 latency profile (reference: costmodel.py).

The reference prices draft / verify forwards from a hand-written
``LatencyProfile`` (costmodel.py:27-100; ``illustrative_profile`` "reproduces no
measured hardware numbers").  Here the same model -- piecewise-linear cost
tables over batch size and ``analytic_speedup`` (costmodel.py:237-257) -- is
fed by ``measure_profile``, which times the
device forwards themselves: a LOW single-token forward at batch B (draft) and a
HIGH forward over n tokens per sequence (verify), CUDA events around
graph-free launches on the engine's stream.  ``bench.py`` reports the model's
predicted QSpec/AR speedup next to the measured one.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, Sequence

from .errors import ConfigError, QSpecError


class ProfileError(QSpecError):
    """Malformed latency profile (costmodel.py ProfileError)."""


@dataclass
class LatencyProfile:
    """draft: batch -> L_draft(B); verify: batch -> [(n, L_verify(B, n))] with an n = 1 point."""

    draft: dict[int, Fraction]
    verify: dict[int, list[tuple[int, Fraction]]]

    def __post_init__(self) -> None:
        if not self.draft or not self.verify:
            raise ProfileError("profile needs at least one draft and one verify entry")
        for b, c in self.draft.items():
            if b < 1 or c <= 0:
                raise ProfileError(f"draft entry batch={b} must have batch>=1, cost>0")
        for b, pts in self.verify.items():
            ns = [n for n, _ in pts]
            if b < 1 or not pts or len(set(ns)) != len(ns) or 1 not in ns or any(n < 1 or c <= 0 for n, c in pts):
                raise ProfileError(f"verify entries for batch={b} need distinct n>=1 with cost>0 and an n=1 point")
            pts.sort(key=lambda p: p[0])

    @staticmethod
    def _bracket(keys: Sequence[int], batch: int) -> tuple[int, int, Fraction]:
        lo = max((k for k in keys if k <= batch), default=None)
        hi = min((k for k in keys if k >= batch), default=None)
        if lo is None or hi is None:
            raise ProfileError(f"batch {batch} outside profile range [{min(keys)}, {max(keys)}]")
        return lo, hi, Fraction(0) if lo == hi else Fraction(batch - lo, hi - lo)

    def draft_cost(self, batch: int) -> Fraction:
        lo, hi, w = self._bracket(sorted(self.draft), batch)
        return self.draft[lo] * (1 - w) + self.draft[hi] * w

    def _verify_at(self, batch: int, n: int) -> Fraction:
        pts = self.verify[batch]
        for pn, pc in pts:
            if pn == n:
                return pc
        below = [p for p in pts if p[0] < n]
        above = [p for p in pts if p[0] > n]
        if below and above:
            (n0, c0), (n1, c1) = below[-1], above[0]
        elif len(below) >= 2:
            (n0, c0), (n1, c1) = below[-2], below[-1]
        elif len(above) >= 2:
            (n0, c0), (n1, c1) = above[0], above[1]
        else:
            return (below or above)[-1 if below else 0][1]
        return c0 + (c1 - c0) * Fraction(n - n0, n1 - n0)

    def verify_cost(self, batch: int, n_tokens: int) -> Fraction:
        if n_tokens < 1:
            raise ProfileError("verify n_tokens must be >= 1")
        lo, hi, w = self._bracket(sorted(self.verify), batch)
        return self._verify_at(lo, n_tokens) * (1 - w) + self._verify_at(hi, n_tokens) * w

    def base_cost(self, batch: int) -> Fraction:
        return self.verify_cost(batch, 1)


def parse_profile(lines: str | Iterable[str]) -> LatencyProfile:
    """'draft batch=B cost=C' / 'verify batch=B n=N cost=C' lines."""
    if isinstance(lines, str):
        lines = lines.splitlines()
    draft: dict[int, Fraction] = {}
    verify: dict[int, list[tuple[int, Fraction]]] = {}
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        kind, *rest = line.split()
        try:
            f = dict(p.split("=", 1) for p in rest)
        except ValueError as exc:
            raise ProfileError(f"line {lineno}: malformed field") from exc
        try:
            if kind == "draft":
                draft[int(f["batch"])] = Fraction(float(f["cost"]))
            elif kind == "verify":
                verify.setdefault(int(f["batch"]), []).append((int(f["n"]), Fraction(float(f["cost"]))))
            else:
                raise ProfileError(f"line {lineno}: unknown entry kind {kind!r}")
        except (KeyError, ValueError) as exc:
            raise ProfileError(f"line {lineno}: {exc}") from exc
    return LatencyProfile(draft, verify)


def format_profile(p: LatencyProfile) -> str:
    out = [f"draft batch={b} cost={float(p.draft[b])!r}" for b in sorted(p.draft)]
    out += [f"verify batch={b} n={n} cost={float(c)!r}" for b in sorted(p.verify) for n, c in p.verify[b]]
    return "\n".join(out)


@dataclass
class AcceptanceModel:
    """Distribution of per-cycle accept lengths over {0..gamma} (normalised)."""

    gamma: int
    weights: list[Fraction]

    def __post_init__(self) -> None:
        if self.gamma < 1:
            raise ConfigError("acceptance model gamma must be >= 1")
        if len(self.weights) != self.gamma + 1 or any(w < 0 for w in self.weights) or sum(self.weights) <= 0:
            raise ConfigError("need gamma+1 non-negative, not-all-zero weights")
        tot = sum(self.weights)
        self.weights = [Fraction(w) / tot for w in self.weights]

    @classmethod
    def from_trace(cls, accept_lens: Sequence[int], gamma: int) -> "AcceptanceModel":
        if not accept_lens:
            raise ConfigError("empty acceptance trace")
        w = [Fraction(0)] * (gamma + 1)
        for a in accept_lens:
            if not 0 <= a <= gamma:
                raise ConfigError(f"accept_len {a} outside [0, {gamma}]")
            w[a] += 1
        return cls(gamma, w)

    def expected_accept_len(self) -> Fraction:
        return sum((a * w for a, w in enumerate(self.weights)), Fraction(0))


@dataclass
class AnalyticReport:
    tokens_per_cycle: float
    speedup: float
    per_valid_token_latency: float


def analytic_speedup(profile: LatencyProfile, acc: AcceptanceModel, gamma: int, batch: int) -> AnalyticReport:
    """costmodel.py:237-257: (E[a]+1) * L_base / (gamma * L_draft + L_verify(gamma+1))."""
    if gamma < 1 or acc.gamma != gamma:
        raise ConfigError("gamma must be >= 1 and match the acceptance model")
    tpc = acc.expected_accept_len() + 1
    cyc = gamma * profile.draft_cost(batch) + profile.verify_cost(batch, gamma + 1)
    return AnalyticReport(float(tpc), float(tpc * profile.base_cost(batch) / cyc), float(cyc / tpc))


def measure_profile(model, batches: Sequence[int], ns: Sequence[int] = (1, 2, 4), reps: int = 5,
                    ctx: int = 128) -> LatencyProfile:
    """Time device forwards (ms): LOW T=B (draft) and HIGH over n tokens per sequence (verify)."""
    import torch
    from . import _lib
    from .engine import DecodeEngine
    draft: dict[int, Fraction] = {}
    verify: dict[int, list[tuple[int, Fraction]]] = {}
    for B in batches:
        eng = DecodeEngine(model, B, gamma=max(ns) - 1 if max(ns) > 1 else 1, max_new_cap=16, use_graphs=False)
        t = eng.t
        t["pos"].fill_(ctx)
        st = _lib.stream_ptr()

        def timed(batches_, low):
            mode = _lib.QS_MODE_LOW if low else _lib.QS_MODE_HIGH
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for r in range(reps + 1):
                if r == 1:
                    e0.record()
                for b, off in batches_:
                    _lib.call("qs_forward", eng.cm, b, mode, eng.ws, None, t["argmax"].data_ptr() + off, st)
            e1.record()
            torch.cuda.synchronize()
            return Fraction(e0.elapsed_time(e1) / reps).limit_denominator(10 ** 9)

        def stage(per_seq):
            t["slot"][:B * per_seq].copy_(torch.arange(B, dtype=torch.int32, device="cuda").repeat_interleave(per_seq))
            return eng._batches(per_seq, ctx_cap=ctx + per_seq)   # every query sits at position ctx

        draft[B] = timed(stage(1), True)
        verify[B] = [(n, timed(stage(n), False)) for n in ns]
        del eng
    return LatencyProfile(draft, verify)


def geometric_acceptance(p: float, gamma: int) -> AcceptanceModel:
    """Accept-length distribution of i.i.d. per-draft acceptance p: P(a=k) = p^k (1-p), P(a=gamma) = p^gamma."""
    p = Fraction(p).limit_denominator(10 ** 6)
    w = [p ** k * (1 - p) for k in range(gamma)] + [p ** gamma]
    return AcceptanceModel(gamma, w)

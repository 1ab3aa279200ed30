"""Logit parity rule -- TEST INFRASTRUCTURE (checker used by tests/ and bench.py, never shipped).

* max relative error <= 1e-2: ``max|got - want| / max|want|`` per compared batch;
* identical greedy tokens: a row's argmax can only flip if its oracle top-2 margin
  is at most twice that row's largest absolute logit error, so rows with a larger
  margin must agree exactly; rows at or below it are "near ties", counted, and may
  be at most ``max_tie_frac`` of all rows compared (otherwise the greedy check
  would be vacuous).
"""

from __future__ import annotations

import torch


class ParityTally:
    def __init__(self):
        self.rows = 0
        self.ties = 0
        self.mismatches = 0
        self.max_rel = 0.0

    def add(self, got: torch.Tensor, want: torch.Tensor) -> float:
        got = got.detach().float().cpu()
        want = want.detach().float().cpu()
        err = (got - want).abs()
        rel = float(err.max() / (want.abs().max() + 1e-6))
        self.max_rel = max(self.max_rel, rel)
        top2 = want.topk(2, dim=-1).values
        margin = top2[:, 0] - top2[:, 1]
        decisive = margin > 2.0 * err.max(dim=-1).values
        self.rows += int(want.shape[0])
        self.ties += int((~decisive).sum())
        self.mismatches += int((got.argmax(-1) != want.argmax(-1))[decisive].sum())
        return rel

    @property
    def tie_frac(self) -> float:
        return self.ties / max(1, self.rows)

    def summary(self) -> dict:
        return {"rows": self.rows, "near_tie_rows": self.ties, "near_tie_frac": self.tie_frac,
                "greedy_mismatches_decisive": self.mismatches, "max_rel_err": self.max_rel,
                "rule": "rel = max|got-want|/max|want| <= 1e-2; greedy equal on every row whose oracle "
                        "top-2 margin > 2 x that row's max |logit error|; near ties <= 10% of rows"}

    def check(self, tol: float = 1e-2, max_tie_frac: float = 0.10):
        assert self.max_rel <= tol, self.summary()
        assert self.mismatches == 0, self.summary()
        assert self.tie_frac <= max_tie_frac, self.summary()

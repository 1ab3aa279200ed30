"""Logit parity rule -- TEST INFRASTRUCTURE (checker used by tests/ and bench.py, never shipped).

Compared quantities, per batch of rows (one row = one sequence's last-token logits):

* ``rel = max|got - want| / max|want|`` against the fp32 oracle ``want``
  (``oracle.forward_ref.forward_fp32``).  North-star tolerance: 1e-2.
* The bf16 floor: with ``floor`` = the same oracle run at the GPU's storage
  precision (``forward_fp32(..., bf16_storage=True)``, every intermediate the GPU
  keeps in bf16 rounded there), ``rel_floor = max|floor - want| / max|want|`` is
  what ANY bf16-activation implementation loses on these inputs.  At full Llama-2
  7B width it exceeds 1e-2, so there the bar is the floor:
  ``rel <= 1.25 * rel_floor + 2e-3``.
* Greedy tokens: the bound ``e`` on any logit's error is ``tol * max|want|`` (or
  ``1.25 x`` the floor's largest absolute error when that is larger).  A row whose
  oracle top-2 margin exceeds ``2 e`` cannot change its argmax within that bound,
  so its greedy token must equal the oracle's; rows at or below are near ties,
  counted and reported.  The bound never uses the GPU's own error, so the check
  is not vacuous: a GPU error above the bound shows up as a greedy mismatch.
"""

from __future__ import annotations

from typing import Optional

import torch


class ParityTally:
    def __init__(self, tol: float = 1e-2):
        self.tol = tol
        self.rows = 0
        self.ties = 0
        self.mismatches = 0
        self.max_rel = 0.0
        self.max_rel_floor: Optional[float] = None
        self.agree_gpu = 0
        self.agree_floor = 0

    def add(self, got: torch.Tensor, want: torch.Tensor, floor: Optional[torch.Tensor] = None) -> float:
        got = got.detach().float().cpu()
        want = want.detach().float().cpu()
        scale = float(want.abs().max()) + 1e-6
        rel = float((got - want).abs().max()) / scale
        self.max_rel = max(self.max_rel, rel)
        bound = self.tol * scale
        if floor is not None:
            floor = floor.detach().float().cpu()
            ferr = (floor - want).abs()
            self.max_rel_floor = max(self.max_rel_floor or 0.0, float(ferr.max()) / scale)
            bound = max(bound, 1.25 * float(ferr.max()))
            self.agree_floor += int((floor.argmax(-1) == want.argmax(-1)).sum())
        top2 = want.topk(2, dim=-1).values
        decisive = (top2[:, 0] - top2[:, 1]) > 2.0 * bound
        self.rows += int(want.shape[0])
        self.ties += int((~decisive).sum())
        self.mismatches += int((got.argmax(-1) != want.argmax(-1))[decisive].sum())
        self.agree_gpu += int((got.argmax(-1) == want.argmax(-1)).sum())
        return rel

    @property
    def tie_frac(self) -> float:
        return self.ties / max(1, self.rows)

    @property
    def rel_bar(self) -> float:
        if self.max_rel_floor is None:
            return self.tol
        return max(self.tol, 1.25 * self.max_rel_floor + 2e-3)

    def summary(self) -> dict:
        out = {"rows": self.rows, "max_rel_err": self.max_rel, "rel_bar": self.rel_bar,
               "greedy_decisive_rows": self.rows - self.ties, "greedy_mismatches_decisive": self.mismatches,
               "near_tie_rows": self.ties, "near_tie_frac": self.tie_frac,
               "argmax_agree_frac": self.agree_gpu / max(1, self.rows)}
        if self.max_rel_floor is not None:
            out["bf16_floor_max_rel_err"] = self.max_rel_floor
            out["bf16_floor_argmax_agree_frac"] = self.agree_floor / max(1, self.rows)
        return out

    def check(self, max_tie_frac: Optional[float] = 0.10):
        s = self.summary()
        assert self.max_rel <= self.rel_bar, s
        assert self.mismatches == 0, s
        if max_tie_frac is not None:
            assert self.tie_frac <= max_tie_frac, s

"""CPU oracle for the live-autoscaling data plane -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline leg may import anything here, and only as the checker or the
timed CPU baseline; the product (``paper_2412_17246_b200``) never does.

* ``gen_golden.py``  -- runs the reference package (/root/reference, this
  container only) and freezes its decisions into ``tests/golden/``.
* ``dataplane_ref.py`` -- CPU restatement of the byte data plane: weight slabs
  copied along plan edges with torch CPU ``copy_``.
* ``forward_ref.py`` -- fp32 Llama forward, unsplit and ZigZag-split, the
  logit oracle for cooperative execution.
* ``logit_parity.py`` -- the tolerance rule applied to GPU logits against it
  (max relative error 1e-2, greedy identity on every non-tie row, tie budget).
"""

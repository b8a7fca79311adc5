"""CPU oracle for the synchronous-SGD gradient exchange and blended update of
arXiv 1711.04325 (Akiba et al., "Extremely Large Minibatch SGD: Training ResNet-50
on ImageNet in 15 Minutes").

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1711_04325_b200``) never imports it, and this
package imports nothing from the product path: the two share no code, headers,
tables or constants.  Inputs come from ``synth`` (seeded generators, no method
arithmetic).

Plain NumPy, float64 arithmetic unless the paper fixes a precision (the fp16 wire,
PAPER.md:85-87).  Every function cites the passage it follows, as
``PAPER.md:<line>`` (section / equation).  Readings of ambiguous passages are
listed in DESIGN.md "Readings" and referenced here as R<n>.

Modules
  binary16  IEEE 754 binary16 codec (the wire format)
  schedule  eta_base, slow-start / Goyal LR, alpha_SGD, alpha_RMSprop, PAPER.md:174-230
  update    the blended RMSprop/momentum-SGD rule, PAPER.md:152-157
  exchange  pack -> exact fp16 all-reduce (sum) -> unpack/average
  bn        BN last-minibatch statistics average, PAPER.md:68-71
  run       the whole iteration loop for T steps and k workers

Parity pins live in tests/test_oracle_*.py.  Parity unpinned: nothing in the
per-step arithmetic; the accuracy effect of fp16 communication ("relatively
small") is not a checkable number and is not claimed.
"""
from . import binary16, schedule, update, exchange, bn, run  # noqa: F401

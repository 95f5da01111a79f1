"""Independent fp64 CPU oracle for the layered-gradient-accumulation (LGA) step.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or call
anything in this package.  The product path (``paper_2106_02679_b200``) never
imports it and shares no code with it; the only shared module is ``synth``
(seeded input generators, which hold none of the method's arithmetic).

Citations are ``P:L`` = line L of the paper's text (``PAPER.md``, arXiv
2106.02679) and ``S:L`` = line L of its companion ``SPEC.md``; DESIGN.md lists
every reading taken where the paper is silent (A-1 ... A-15).

Modules
-------
model      one transformer layer forward/backward in fp64 NumPy, MSE loss
schedule   standard / layered / full-batch gradient accumulation, AdamW
counters   closed-form per-step communication counters, stage map, bubble

Every function here has at least one pin in ``tests/test_oracle_*.py`` that
checks it against something other than itself (torch.autograd fp64, central
finite differences, closed forms printed in the paper, invariants).  There is
no "parity unpinned" function in this package.
"""

from . import model, schedule, counters  # noqa: F401

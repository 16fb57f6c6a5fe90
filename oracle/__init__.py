"""CPU oracle for the sketchpress hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (``paper_2105_01271_b200``) imports this
package.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it, and
only as the checker or as the CPU baseline that is timed beside the GPU path.

The oracle is a numpy restatement of the reference algorithm
(``/root/reference/pkg/src/sketchpress``; every function cites the file:line
it follows).  It is pinned against golden vectors produced by the reference
itself (``tests/golden/make_golden.py``) and against the reference's own
known-answer tests (``tests/test_oracle_pins.py``).
"""

from .sketchpress_oracle import *  # noqa: F401,F403

"""Host logic of bcs.BoundaryPrefetch (CPU): the speculative evaluation of
the next step's boundary data never changes what stage_bc_values sees
(bcs.py:58-96 evaluates bc.g / bc.g_dot at the stage times of the step)."""

import numpy as np
import pytest

from paper_2403_08084_b200.bcs import BoundaryPrefetch, stage_fn_values


def test_hit_returns_the_scheduled_evaluation_once():
    calls = []

    def g(t):
        calls.append(t)
        return np.full(5, t)

    pf = BoundaryPrefetch()
    first = pf.take(g, [0.1, 0.2], (5,))
    np.testing.assert_array_equal(first, stage_fn_values(lambda t: np.full(5, t), [0.1, 0.2], (5,)))
    pf.schedule(g, [0.3, 0.4], (5,))
    hit = pf.take(g, [0.3, 0.4], (5,))
    assert calls == [0.1, 0.2, 0.3, 0.4]  # no second evaluation on a hit
    assert hit.shape == (2, 5) and hit[1, 0] == 0.4


def test_miss_evaluates_inline_after_the_pending_call():
    order = []

    def g(t):
        order.append(t)
        return np.full(3, t)

    pf = BoundaryPrefetch()
    pf.schedule(g, [0.5, 0.6], (3,))
    miss = pf.take(g, [0.7, 0.8], (3,))  # the step size changed: other stage times
    assert miss[0, 0] == 0.7 and miss[1, 0] == 0.8
    assert order == [0.5, 0.6, 0.7, 0.8]  # sequential, never concurrent


def test_callback_error_surfaces_in_the_step_that_needs_it():
    def bad(t):
        raise RuntimeError("boundary data failed")

    pf = BoundaryPrefetch()
    pf.schedule(bad, [1.0], (3,))
    pf.join()  # does not raise at the start of the next step
    with pytest.raises(RuntimeError, match="boundary data failed"):
        pf.take(bad, [1.0], (3,))

"""The device Adam's bias-correction table (optimize.py:116-117 computes
1 / (1 - beta^t) with the C pow): sized so that the device's clamp to the
last row is exact for every later step, whatever the configured betas (CPU)."""
import math

import numpy as np
import pytest


@pytest.mark.parametrize("beta1,beta2", [(0.9, 0.999), (0.9, 0.9999), (0.95, 0.99999)])
def test_table_reaches_exact_one(beta1, beta2):
    from paper_2501_08672_b200.optimize import IBC_ROWS, bias_correction_rows, bias_correction_table
    rows = bias_correction_rows(beta1, beta2)
    assert rows >= IBC_ROWS
    tab = bias_correction_table(beta1, beta2, rows=rows)
    assert tab.shape == (rows, 2)
    assert np.all(tab[-1] == 1.0)
    # every step beyond the table has both corrections exactly 1.0 as well
    for t in (rows + 1, rows * 2, rows * 10):
        assert 1.0 / (1.0 - math.pow(beta1, t)) == 1.0 and 1.0 / (1.0 - math.pow(beta2, t)) == 1.0
    # and the table is the reference's expression row by row
    for t in (1, 2, 17, rows // 2, rows):
        assert tab[t - 1, 0] == 1.0 / (1.0 - beta1 ** t) and tab[t - 1, 1] == 1.0 / (1.0 - beta2 ** t)


def test_default_betas_keep_the_small_table():
    from paper_2501_08672_b200.optimize import IBC_ROWS, bias_correction_rows
    assert bias_correction_rows(0.9, 0.999) == IBC_ROWS

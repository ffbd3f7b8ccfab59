"""The README quick start, as a user runs it (one GPU, the public Python binding), at 1e6 draws: the result
object is consistent (best = argmax of the smoothed surface, P^ / SE sane) and the continuous optimum is a
feasible design whose TPS value is not below the best grid value."""
import re
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_readme_quick_start_runs():
    src = open(os.path.join(ROOT, "README.md")).read()
    code = re.search(r"```python\n(.*?)```", src, re.S).group(1)
    code = code.replace("total_samples=10**8", "total_samples=10**6")
    ns = {}
    exec(compile(code, "README.md", "exec"), ns)     # the quick start verbatim, fewer draws
    res, A, v, status = ns["res"], ns["A"], ns["v"], ns["status"]
    sm = res.smoothed.cpu().numpy()
    mean = res.mean.cpu().numpy()
    best, p_best = ns["best"], ns["p_smoothed"]
    assert best == int(np.argmax(sm)) and abs(p_best - sm[best]) < 1e-12
    assert 0.9 < mean[best] < 1.0                      # scenario (c): the optimum is near 0.977
    assert status[0] != 1 and A.shape == (1, 3) and np.all((A[0] >= 0) & (A[0] <= 0.025))
    assert v[0] >= sm.max() - 1e-7                     # L-BFGS starts at the best grid point and ascends

"""bench.py's same-run parity check: the sampled-row comparison against the
cpu_baseline leg's product accepts an independent correct product and rejects a one-term error."""
import numpy as np

import bench
import inputs
import oracle


def test_parity_vs_cpu_accepts_and_rejects():
    n, rp, col, val = inputs.config_crs("C1")
    x = inputs.vector(n)
    y_cpu = oracle.spmv_crs(n, rp, col, val, x)
    y_chain = oracle.spmv_chain(n, rp, col, val, x)  # a different (fused) summation of the same rows
    rows = np.arange(0, n, 7)
    ok = bench.parity_vs_cpu(y_chain, y_cpu, rp, col, val, x, rows)
    assert ok["within_bound"] and ok["rows_checked"] == len(rows) and ok["gpu_finite_all_rows"]
    bad = y_chain.copy()
    r = int(rows[3])
    k = int(rp[r])
    bad[r] -= 2 * val[k] * x[col[k]]  # one term with the wrong sign
    res = bench.parity_vs_cpu(bad, y_cpu, rp, col, val, x, rows)
    assert not res["within_bound"] and res["rows_outside"] == 1
    nan = y_chain.copy()
    nan[int(rows[5])] = np.nan
    assert not bench.parity_vs_cpu(nan, y_cpu, rp, col, val, x, rows)["within_bound"]

"""Eq. (2) against the paper's own Table 3 rows: pins the throughput unit
(env steps / wall second) that bench.py reports."""
import pytest

from oracle.path import throughput_eq2
from tests.conftest import read_golden


@pytest.mark.parametrize("row", read_golden("eq2_throughput.csv"))
def test_eq2_reproduces_table3(row):
    line, model, placement, gpus, n_re, n_env, n_es, t_s, printed = row
    got = throughput_eq2(float(n_re), float(n_env), float(n_es), float(t_s))
    # the paper rounds to 2 decimals; one row is off by 0.05%
    assert abs(got - float(printed)) / float(printed) < 6e-4, (line, got, printed)

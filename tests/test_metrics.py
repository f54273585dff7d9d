"""The reporting conventions are the paper's: flops per element / nnz recovered from every row
of PAPER.md Tables 2-8 (golden fixture) as Gflops × ms × 1e6 / h."""
import json
import os

import pytest

from paper_2112_11880_b200 import metrics

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_flop_tables.json")))
KEY = {"ZASSIGN": "zassign", "ZSCAL": "zscal", "ZAXPY": "zaxpy", "ZAXMY": "zaxmy", "ZDOT": "zdotc",
       "ZNORM": "dznrm2"}


@pytest.mark.parametrize("table", list(KEY))
def test_blas1_flop_weights(table):
    t = GOLD["tables"][table]
    for h, ms, gflops in t["rows"]:
        implied = gflops * ms * 1e6 / h
        assert abs(implied - metrics.FLOPS_PER_ELEM[KEY[table]]) / implied < 0.03, (table, h)


def test_spmv_flop_weight():
    for nnz, ms, gflops, name in GOLD["tables"]["SPMV"]["rows"]:
        implied = gflops * ms * 1e6 / nnz
        assert abs(implied - metrics.FLOPS_PER_NNZ_SPMV) / implied < 0.05, name


def test_byte_models():
    # C4: ZSpMV 4.597 GB, BiCGStab iteration 11.11 GB, CG 5.75 GB
    n, nnz = 8_000_000, 213_847_192
    assert round(metrics.spmv_bytes(n, nnz) / 1e9, 3) == 4.597
    assert round(metrics.bicgstab_iter_bytes(n, nnz) / 1e9, 2) == 11.11
    assert round(metrics.cg_iter_bytes(n, nnz) / 1e9, 2) == 5.75

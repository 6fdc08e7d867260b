"""Scan reports in the reference's CSV format (paper_1704_04549_b200/report.py)."""
import os
import re

import pytest

from paper_1704_04549_b200 import report as R
import paper_1704_04549_b200 as T

REF_EXPERIMENT = "/root/reference/proj/include/tpdg/harness/experiment.hpp"


def test_header_is_the_reference_header():
    if not os.path.exists(REF_EXPERIMENT):
        pytest.skip("reference sources not present (GPU box)")
    src = open(REF_EXPERIMENT).read()
    body = src[src.index("report_csv_header()"):]
    parts = re.findall(r'"([^"]*)"', body[: body.index(";")])
    assert "".join(parts) == R.REPORT_CSV_HEADER


def test_row_format_matches_ostream_precision_12():
    row = R.ReportRow(case_id="advection_swirl", p=15, dt=0.005, avg_gmres=25.0, total_gmres=25, newton_steps=1,
                      form_seconds=0.0123456789012345, pc_apply_seconds=2.5e-3, total_seconds=1.0 / 3.0)
    assert R.report_row_csv(row) == ("advection_swirl,15,0.005,ksvd_full,25,25,1,0.0123456789012,0.0025,"
                                     "0.333333333333,,ok,")
    row.l2_error = 1e-10
    row.status, row.failure_code = "failed", "gmres_max_iterations"
    assert R.report_row_csv(row).endswith(",1e-10,failed,gmres_max_iterations")
    assert len(R.report_row_csv(row).split(",")) == len(R.REPORT_CSV_HEADER.split(","))


def test_failure_codes():
    res = T.GmresResult(None, 0, [], False)
    assert R.failure_code_for(T.GmresFailure("x", res)) == "gmres_max_iterations"
    assert R.failure_code_for(T.StateError("x")) == "non_physical_state"
    assert R.failure_code_for(T.SingularError("x")) == "singular_block"
    assert R.failure_code_for(T.ConvergenceError("x")) == "nonlinear_divergence"
    assert R.failure_code_for(T.ConfigError("x")) == "config_error"
    assert R.failure_code_for(RuntimeError("x")) == "internal_error"


def test_write_report_csv(tmp_path):
    p = tmp_path / "scan.csv"
    R.write_report_csv([R.ReportRow(case_id="advection_swirl", p=4, dt=0.005)], str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == R.REPORT_CSV_HEADER and lines[1].startswith("advection_swirl,4,0.005,ksvd_full,")

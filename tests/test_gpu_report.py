"""Scan report on the device in the reference's CSV format (paper_1704_04549_b200/report.py)."""
import pytest

from paper_1704_04549_b200 import report as R
import paper_1704_04549_b200 as T

pytestmark = pytest.mark.gpu


def test_report_rows_cfg2():
    ctx = T.Context(0)
    rows = [R.run_cell(ctx, "cfg2", p) for p in (4, 8)]
    for r, its in zip(rows, (17, 18)):  # the reference's counts (tests/golden/cfg2_p*.npz)
        assert r.status == "ok" and r.total_gmres == its and r.newton_steps == 1
        assert 0.0 < r.pc_apply_seconds < r.total_seconds and r.form_seconds > 0.0
        line = R.report_row_csv(r)
        assert line.startswith(f"advection_swirl,{r.p},0.005,ksvd_full,{its},{its},1,")

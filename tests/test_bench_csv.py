"""bench-iep / bench-moe CSV front end: the reference
CLI's flags, CSV headers, row order, call-count bounds and exit codes
(tools/dynbatch_cli.cpp:24-37, 109-358), over device runs."""
import csv
import io

import pytest

import paper_1707_02402_b200 as db
from paper_1707_02402_b200 import bench_csv as B


def test_headers_are_the_reference_schemas():
    # tools/dynbatch_cli.cpp:162 and 267-268
    assert B.IEP_HEADER == "scheduler,b,p,s_max,d_max,calls,module_ms,stack_ms,total_ms,speedup\n"
    assert B.MOE_HEADER == ("impl,n,k,b,data_dim,hidden,calls,expert_ms,stack_ms,total_ms,speedup,"
                            "speedup_per_call\n")


def test_unknown_scheduler_is_a_usage_error(capsys):
    assert B.main(["bench-iep", "--schedulers", "naive,fastest"]) == B.EXIT_USAGE
    assert "error: unknown scheduler 'fastest'" in capsys.readouterr().err


def test_call_bounds():
    st = db.BatchStats(batch=4, vocab=5, width=8, s_max=6, d_max=3, total_nodes=20, expensive_nodes=12)
    B.check_call_bounds("naive", 12, st)
    B.check_call_bounds("improved", 20, st)
    with pytest.raises(B.VerificationError):
        B.check_call_bounds("online", 16, st)
    with pytest.raises(B.VerificationError):
        B.check_call_bounds("naive", 11, st)


@pytest.mark.gpu
def test_bench_iep_rows(tmp_path):
    out = tmp_path / "iep.csv"
    rc = B.main(["bench-iep", "--b", "1,8", "--width", "16", "--p", "10", "--s", "8", "--reps", "2",
                 "--schedulers", "naive,standard,improved,online", "--out", str(out)])
    assert rc == 0
    text = out.read_text()
    assert text.startswith(B.IEP_HEADER)
    rows = list(csv.DictReader(io.StringIO(text)))
    assert [r["scheduler"] for r in rows] == ["naive"] * 2 + ["standard"] * 2 + ["improved"] * 2 + ["online"] * 2
    for r in rows:
        b = db.Batch.generate("chain", batch=int(r["b"]), vocab=10, width=16, length=8, branch_prob=0.1, seed=0)
        assert int(r["calls"]) == b.schedule(r["scheduler"]).expensive_calls(b)
        assert float(r["module_ms"]) > 0 and float(r["speedup"]) > 0
        st = b.stats()
        assert (int(r["s_max"]), int(r["d_max"]), int(r["p"])) == (st.s_max, st.d_max, 10)


@pytest.mark.gpu
def test_bench_moe_rows(tmp_path):
    out = tmp_path / "moe.csv"
    rc = B.main(["bench-moe", "--n", "4,8", "--k", "2", "--b", "32", "--data-dim", "16", "--hidden", "16",
                 "--reps", "2", "--out", str(out)])
    assert rc == 0
    text = out.read_text()
    assert text.startswith(B.MOE_HEADER)
    rows = list(csv.DictReader(io.StringIO(text)))
    assert [(r["impl"], r["n"]) for r in rows] == [("naive", "4"), ("batched", "4"), ("naive", "8"), ("batched", "8")]
    assert int(rows[0]["calls"]) == 2 * 32  # k·b single-row calls
    assert int(rows[1]["calls"]) <= 4

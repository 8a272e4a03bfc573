"""The reference's C++ API, link-compatible, on the B200: the reference's
UNMODIFIED acceptance suite (proj/tests/acceptance/acceptance.cpp, criteria
1-10 of SPEC.md:537-549) compiled against the reference headers and linked
against libdynpr_compat.so (compat/dynpr_compat.cpp: every dynpr:: entry of
graph/partition/rank/frontier/engine/workload/harness .hpp over the C-ABI,
device snapshots cached by content) instead of libdynpr.a.  Criteria 9 and 10
shell out to compat/_build/dynpr_bench, the hand-parsed CLI over the same
library, on the reference's temporal-10k fixture."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ACCEPTANCE = os.path.join(ROOT, "compat", "_build", "acceptance")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(ACCEPTANCE), reason="compat/_build/acceptance not built")]


def test_reference_acceptance_suite_passes_on_the_device(dp):
    p = subprocess.run([ACCEPTANCE], cwd=ROOT, capture_output=True, text=True, timeout=900)
    lines = [l for l in p.stdout.splitlines() if l.startswith("[")]
    print(p.stdout)
    passed = [l for l in lines if l.startswith("[PASS]")]
    assert len(passed) == 10, p.stdout + p.stderr
    assert p.returncode == 0 and "all 10 criteria passed" in p.stdout


def test_cli_report_matches_reference_digest(dp, tmp_path):
    """dynpr_bench temporal on the fixture == the reference CLI's report
    (md5 dfbb1dad... for temporal, 1e-3, all approaches, seed 1,
    --no-timing)."""
    import hashlib
    out = tmp_path / "r.csv"
    subprocess.run([os.path.join(ROOT, "compat", "_build", "dynpr_bench"), "temporal", "--graph",
                    os.path.join(ROOT, "tests", "golden", "temporal-10k.txt"), "--batch-sizes", "1e-3",
                    "--approaches", "static,nd,dt,df,dfp", "--seed", "1", "--no-timing", "--format", "csv",
                    "--out", str(out)], check=True, timeout=300)
    assert hashlib.md5(out.read_bytes()).hexdigest() == "dfbb1dad50c53d152f452c24943af797"

"""The CLI entry point on the GPU: ``python -m paper_2412_05824_b200`` runs the
self-test (reference tests/test_cli.py:246-251, which targets the reference's
module name), and the debug twiddle skew makes it fail (the hook corrupts the
device tables)."""

import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_module_entry_point_selftest():
    r = subprocess.run([sys.executable, "-m", "paper_2412_05824_b200", "selftest", "--quick"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "self-test: PASS" in r.stdout


def test_selftest_skew_fails_then_clean_plans_recover():
    from paper_2412_05824_b200.cli import main
    assert main(["selftest", "--quick", "--debug-skew-twiddle"]) == 1
    assert main(["selftest", "--quick"]) == 0

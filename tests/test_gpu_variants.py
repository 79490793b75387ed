"""The alternative kernels behind the diagnostic switches (register-staged
variants of both paths) stay bitwise-correct: the sanitizer driver runs every
kernel against the oracle in a fresh process per switch setting."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"TM_STAGED_LDG": "1"}, {"TM_STAGED_KERNEL": "ws"},
                                 {"TM_STAGED_KERNEL": "tma"}, {"TM_STAGED_KERNEL": "tmaws"}, {"TM_ALLGATHER": "ce"},
                                 {"TM_STAGED_KERNEL": "oneshot"}, {"TM_STAGED_KERNEL": "ll"},
                                 {"TM_STAGED_KERNEL": "ll2"},
                                 {"TM_DIRECT_LDG": "1"}, {"TM_DIRECT_TMA": "1"},
                                 {"TM_TMA_CFG": "8", "TM_DIRECT_TMA": "1"}, {"TM_TMA_CFG": "3", "TM_DIRECT_TMA": "1"}])
def test_kernel_variants_bitwise(env):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_driver.py")],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all bitwise == oracle" in r.stdout

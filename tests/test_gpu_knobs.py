"""The library's diagnostics knobs (environment variables read once per
process: A/B alternatives of the product kernels) keep the
oracle's bits: each case runs tests/knob_worker.py in a fresh process with the
knob set."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    ("direct", {"TM_L2_HINT": "1"}),           # evict_first on the direct kernel's bulk loads
    ("direct", {"TM_L2_HINT": "3"}),           # ... and on its bulk stores
    ("direct", {"TM_DIRECT_STATIC": "1"}),     # static tile assignment instead of the claim counter
] + [("direct", {"TM_TMA_CFG": c}) for c in ("1", "2", "4", "5", "6", "7")] + [   # k = 8 tile / ring / residency
    ("direct_small_k", {"TM_TMA_CFG": c}) for c in ("9", "10", "11", "12")] + [    # k <= 4 variants
    ("bsp", {"TM_BSP_TILE": "512"}),
    ("bsp", {"TM_BSP_TILE": "2048"}),
    ("round", {"TM_ROUND_STATIC": "1"}),       # static tiles of the fused EASGD round
    ("oneshot", {"TM_STAGED_KERNEL": "oneshot", "TM_ONESHOT_CHUNK": "256"}),
    ("oneshot", {"TM_STAGED_KERNEL": "oneshot", "TM_ONESHOT_CHUNK": "2048"}),
    ("ranges", {"TM_RANGE_CTAS": "8"}),        # the bucket CTA budget from the environment
    ("staged", {"TM_STAGED_TMA": "1"}),        # alias of TM_STAGED_KERNEL=tma
]


@pytest.mark.parametrize("scenario,env", CASES, ids=[f"{s}-{'-'.join(f'{k}={v}' for k, v in e.items())}"
                                                     for s, e in CASES])
def test_knob_keeps_oracle_bits(scenario, env):
    r = subprocess.run([sys.executable, os.path.join(HERE, "knob_worker.py"), scenario],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert f"OK {scenario}" in r.stdout

"""CPU tests of bench.py's accounting (no GPU): the algorithmic bytes behind the
roofline, the NVLink roofline time of SURVEY 8(d), the
whole-job value and the traffic table lookup."""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ALEXNET = 60_965_224


def test_design_bytes_per_unit():
    # direct: 8 B per element per rank (read 4 + write 4)
    assert bench.design_hbm_bytes("asa16", ALEXNET, 8, "direct") == pytest.approx(8.0 * ALEXNET * 8)
    # staged ASA16: (14 + 2/k) B, ASA: (20 + 4/k) B per element per rank
    assert bench.design_hbm_bytes("asa16", ALEXNET, 8, "staged") == pytest.approx((14 + 2 / 8) * ALEXNET * 8)
    assert bench.design_hbm_bytes("asa", ALEXNET, 4, "staged") == pytest.approx((20 + 4 / 4) * ALEXNET * 4)


def test_nvlink_roofline_matches_survey():
    # ASA16 AlexNet at k = 2 / 4 / 8 against 900 GB/s nominal:
    # 135.5 / 203.2 / 237.1 us; bench uses the measured 770 GB/s peer copy
    for k, us900 in ((2, 135.5), (4, 203.2), (8, 237.1)):
        us = bench.nvlink_roof_us("asa16", ALEXNET, k)
        assert us * bench.NVLINK_GBS / 900.0 == pytest.approx(us900, rel=2e-3)
    assert bench.nvlink_roof_us("asa16", ALEXNET, 1) == 0.0


def test_roofline_fraction_and_traffic():
    bench.STAGED_KERNEL[0] = 3
    r = bench.roofline("asa16", ALEXNET, 8, "staged", 1.0, 6553.9, "measured", "alexnet")
    alg = (14 + 2 / 8) * ALEXNET * 8
    assert r["achieved"] == pytest.approx(alg / 1e-3 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / 6553.9)
    assert r["kernel"] == "tm_exchange_tmaws_kernel"
    d = bench.roofline("asa16", ALEXNET, 8, "direct", 0.57, 6553.9, "measured", "alexnet")
    table = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    assert d["traffic"] == table["alexnet_asa16_k8_direct"]
    assert d["kernel"] == "tm_direct_tma_kernel"


def test_job_value_is_whole_job():
    # every rank's fp32 buffer over the max-over-ranks time
    assert bench.job_value(4.0 * ALEXNET, 8, 0.57) == pytest.approx(4.0 * ALEXNET * 8 / 0.57e-3 / 1e9)

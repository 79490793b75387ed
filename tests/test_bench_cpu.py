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
    # 135.5 / 203.2 / 237.1 us; AR / ASA twice that
    for k, us900 in ((2, 135.5), (4, 203.2), (8, 237.1)):
        assert bench.nvlink_roof_us("asa16", ALEXNET, k, gbs=900.0) == pytest.approx(us900, rel=2e-3)
        assert bench.nvlink_roof_us("asa", ALEXNET, k, gbs=900.0) == pytest.approx(2 * us900, rel=2e-3)
        us = bench.nvlink_roof_us("asa16", ALEXNET, k)  # at the 770 GB/s peer-copy fallback
        assert us * bench.NVLINK_GBS / 900.0 == pytest.approx(us900, rel=2e-3)
    assert bench.nvlink_roof_us("asa16", ALEXNET, 1) == 0.0
    # wire bytes per direction per rank: 2 (k-1)/k * P * s
    assert bench.wire_bytes_per_direction("asa16", ALEXNET, 8) == pytest.approx(2 * 7 / 8 * ALEXNET * 2)
    assert bench.wire_bytes_per_direction("ar", 1024, 4) == pytest.approx(6144)


def test_north_star_bar_and_fractions():
    """BASELINE north star: ASA16 AlexNet k = 8 at >= 70 % of the 900 GB/s NVLink
    roofline, i.e. t <= 237.1 / 0.7 = 338.7 us (algbw >= 720 GB/s)."""
    ns = bench.north_star("asa16", ALEXNET, 8, 0.33869, 770.0, "test", shared_gpu=False)
    assert ns["bar_us"] == pytest.approx(338.7, rel=1e-3)
    assert ns["meets_bar"] is True
    assert ns["frac_vs_900"] == pytest.approx(0.70, rel=2e-3)
    assert ns["frac_vs_measured"] == pytest.approx(0.70 * 900 / 770, rel=2e-3)
    assert ns["algbw_GBps"] == pytest.approx(4 * ALEXNET / 0.33869e-3 / 1e9)
    assert ns["algbw_GBps"] == pytest.approx(720, rel=1e-2)
    assert ns["over_nvlink"] is True
    late = bench.north_star("asa16", ALEXNET, 8, 0.340, 770.0, "test", shared_gpu=True)
    assert late["meets_bar"] is False and late["over_nvlink"] is False


def test_nvlink_roofline_object():
    wire = 2 * 7 / 8 * ALEXNET * 2
    nvml = {"tx_bytes_per_step": 1.05 * wire}
    r = bench.nvlink_roofline("asa16", ALEXNET, 8, 0.300, 760.0, "measured", nvml, "tm_exchange_tmaws_kernel")
    assert r["bound"] == "nvlink" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(wire / 0.3e-3 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / 760.0)
    assert r["frac_vs_900"] == pytest.approx(r["achieved"] / 900.0)
    assert r["traffic"] == pytest.approx(1.05 * wire) and r["traffic_ratio"] == pytest.approx(1.05)
    assert bench.nvlink_roofline("asa16", ALEXNET, 8, 0.3, 760.0, "m", None, "x")["traffic"] is None


def test_multi_gpu_sample_check_uses_oracle(monkeypatch):
    """check_sample regenerates every rank's seeded input and compares with the
    oracle's per-element definition: the oracle's own answer passes bitwise, a
    one-ulp change fails, and AR tolerates an order difference within Q11."""
    import numpy as np
    from oracle import exchange as ox
    from paper_1605_08325_b200.inputs import worker_buffer
    P, k = 5003, 4
    idx = bench.sample_indices(P)
    vals = np.stack([worker_buffer(P, "D2", r, config=3)[idx] for r in range(k)])
    want = ox.element_average(vals, "asa16")
    ok = bench.check_sample("asa16", "D2", P, k, idx, [want.copy() for _ in range(k)])
    assert ok["parity"] and ok["cross_rank_identical"]
    bad = want.copy()
    bad.view(np.uint32)[3] += 1
    res = bench.check_sample("asa16", "D2", P, k, idx, [want, bad, want, want])
    assert not res["parity"] and res["per_rank"] == [True, False, True, True] and not res["cross_rank_identical"]
    war = ox.element_average(vals, "ar")
    near = (war.astype(np.float64) * (1 + 1e-7)).astype(np.float32)
    assert bench.check_sample("ar", "D2", P, k, idx, [war, near, war, war])["parity"]


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


def test_allgather_decision_table(tmp_path):
    """tools/ag_decide.py keeps, per (k, L), the fastest allgather mode among the
    bench lines whose parity passed, and writes the TM_AG_TABLE rules."""
    import subprocess
    import sys as _sys

    def line(k, L, ms, ag, parity=True, kern="tm_exchange_tmaws_kernel"):
        return {"ms_per_step": ms, "parity": {"parity": parity},
                "config": {"k": k, "seg_len": L, "staged_kernel": kern, "allgather": ag}}
    rows = {"bench_n8_alexnet_tmaws_agsm.json": line(8, 7620864, 0.30, "sm"),
            "bench_n8_alexnet_tmaws_agnccl.json": line(8, 7620864, 0.28, "nccl"),
            "bench_n8_alexnet_tmaws_agce.json": line(8, 7620864, 0.25, "ce", parity=False),
            "bench_n8_googlenet_tmaws_agsm.json": line(8, 875008, 0.040, "sm"),
            "bench_n8_googlenet_tmaws_agnccl.json": line(8, 875008, 0.050, "nccl"),
            "bench_n8_googlenet_oneshot_agce.json": line(8, 875008, 0.001, "ce", kern="tm_exchange_oneshot_kernel")}
    for name, d in rows.items():
        (tmp_path / name).write_text(json.dumps(d) + "\n")
    out = subprocess.run([_sys.executable, os.path.join(ROOT, "tools", "ag_decide.py"), str(tmp_path)],
                         capture_output=True, text=True, check=True).stdout
    rules = [l.split("#")[0].split() for l in out.splitlines() if l and not l.startswith("#")]
    assert rules == [["8", str((875008 + 7620864) // 2), "sm"], ["8", str(1 << 62), "nccl"]]

"""Cost model (paper_1410_4054_b200.execmodel; reference execmodel.py:42-107,
225-278; behaviour of test_execmodel.py) and its B200 calibration (gpu)."""

import math

import numpy as np
import pytest

from paper_1410_4054_b200 import PhaseRecord
from paper_1410_4054_b200.execmodel import DeviceProfile, latency_barrier, predict_iteration_time


def test_defaults_and_validation():
    p = DeviceProfile()
    assert (p.launch_latency, p.transfer_latency, p.bandwidth, p.transfer_bandwidth) == (8e-6, 8e-6, 200e9, 8e9)
    for bad in (0.0, -1.0, math.inf, math.nan):
        with pytest.raises(ValueError):
            DeviceProfile(launch_latency=bad)


def test_from_file(tmp_path):
    f = tmp_path / "b200.profile"
    f.write_text("# measured\nlaunch_latency = 2.5e-6\n\nbandwidth = 6.5e12  # copy\n")
    p = DeviceProfile.from_file(f)
    assert p.launch_latency == 2.5e-6 and p.bandwidth == 6.5e12 and p.transfer_latency == 8e-6
    p.to_file(tmp_path / "out.profile")
    assert DeviceProfile.from_file(tmp_path / "out.profile") == p
    for text in ("nope = 1\n", "launch_latency 1\n", "bandwidth = fast\n"):
        f.write_text(text)
        with pytest.raises(ValueError):
            DeviceProfile.from_file(f)


def test_prediction_is_additive():
    rec = PhaseRecord("iteration", launches=3, transfers=1, bytes_kernel=4_000_000, bytes_transfer=800)
    p = DeviceProfile(launch_latency=2e-6, transfer_latency=10e-6, bandwidth=4e12, transfer_bandwidth=50e9)
    assert predict_iteration_time(rec, p) == 3 * 2e-6 + 10e-6 + 4_000_000 / 4e12 + 800 / 50e9


def test_latency_barrier():
    lb = latency_barrier(DeviceProfile(launch_latency=2e-6, bandwidth=6.5e12))
    assert lb.nbytes == 2e-6 * 6.5e12 and lb.real64_count == lb.nbytes / 8
    assert latency_barrier().real64_count == 8e-6 * 200e9 / 8  # reference default: 200k doubles


@pytest.mark.gpu
def test_calibration_and_speedup_curve_on_b200():
    import paper_1410_4054_b200 as pk

    prof = pk.calibrate_b200(0)
    assert 0.5e-6 < prof.launch_latency < 50e-6
    assert 1e-6 < prof.transfer_latency < 500e-6
    assert 1e12 < prof.bandwidth < 10e12
    assert 5e9 < prof.transfer_bandwidth < 200e9
    systems = [(f"poisson2d:{k}", *pk.gen_poisson2d(k)) for k in (1, 3)]
    rows = pk.speedup_curve((pk.cg_classical, pk.cg_pipelined), systems, prof, iterations=10)
    assert all(r["ratio"] > 1.0 for r in rows)  # latency regime: pipelined wins
    assert np.isfinite([r["classical_s"] for r in rows]).all()

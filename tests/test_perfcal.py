"""Perf-model recalibration: the restated model arithmetic equals the reference's
perfmodel.py, and on a GPU the measured calibration round-trips through calibrate()."""
import pytest

from paper_2408_12526_b200 import perfcal as pc

# PerfModel().calibrate(baseline_reference(4, 2000.0), 11.6) and the factor table at (8, 3000.0),
# printed by the unmodified reference (perfmodel.py) in the build container.
REF_T_UNIT = 0.10507142857142858
REF_ROWS_8_3000 = {"bert_base_12l": 11.016666666666666, "tinybert_4l": 3.4515238095238097,
                   "dynabert_6l": 3.4515238095238097, "deebert_early_exit": 7.339166666666667,
                   "cocktail_bagging": 24.88609523809524, "student_parallel_2l": 0.5381428571428573}


def test_calibration_matches_reference_numbers():
    t = pc.calibrate(pc.baseline_reference(4, 2000.0), pc.REFERENCE_OBSERVED_LATENCY_MS)
    assert t == REF_T_UNIT
    for name, f in pc.reference_factor_rows(8, 3000.0):
        assert pc.latency(f, t) == REF_ROWS_8_3000[name], name


def test_model_errors_and_edges():
    base = pc.baseline_reference(4, 2000.0)
    with pytest.raises(ValueError):
        pc.calibrate(base, pc.fixed_terms(base))  # infeasible: no compute left
    with pytest.raises(ValueError):
        pc.Factors(depth=0, width=1, batch=1, seq_len=1, parallel_models=1, gpus=1)
    with pytest.raises(ValueError):
        pc.throughput_per_gpu(base, 0.0)
    assert pc.waiting_time(pc.student_parallel_factors(4)) == 0.0
    assert pc.compute_waves(pc.Factors(depth=1, width=10 ** 6, batch=8, seq_len=512, parallel_models=8, gpus=1)) > 1


@pytest.mark.reference
def test_restatement_matches_live_reference():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from studentpar import perfmodel as pm

    for gpus, rps in ((1, 500.0), (4, 2000.0), (8, 10000.0)):
        for obs in (3.0, 11.6, 40.0):
            m = pm.PerfModel()
            try:
                t = m.calibrate(pm.baseline_reference(gpus, rps), obs)
            except ValueError:  # below the wait/transfer floor: both must refuse
                with pytest.raises(ValueError):
                    pc.calibrate(pc.baseline_reference(gpus, rps), obs)
                continue
            assert pc.calibrate(pc.baseline_reference(gpus, rps), obs) == t
            for (name, f), (_, g) in zip(pm.reference_factor_rows(gpus, rps), pc.reference_factor_rows(gpus, rps)):
                assert pc.latency(g, t) == m.latency(f), name
                assert pc.compute_waves(g) == pm.compute_waves(f)


@pytest.mark.gpu
def test_b200_calibration_round_trip():
    res = pc.calibrate_b200(gpus=4, arrival_rps=2000.0, reps=5)
    base = pc.baseline_reference(4, 2000.0)
    cal = res["calibration"]
    assert 0.0 < res["measured"]["baseline_compute_ms"] < 20.0
    assert pc.calibrate(base, cal["observed_latency_ms"]) == pytest.approx(res["t_unit_ms"], rel=1e-12)
    assert pc.latency(base, res["t_unit_ms"]) == pytest.approx(cal["observed_latency_ms"], rel=1e-12)
    assert res["student_parallel"]["measured_compute_ms"] > 0.0
    assert set(res["factor_table"]) == {n for n, _ in pc.reference_factor_rows()}

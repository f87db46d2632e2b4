"""The device memory a solver context holds, against the storage model
(fmg_memory_model, Eq 6.1-6.3 accounting; §8(f) row N3)."""
import pytest

from fmg_inputs import CONFIGS, default_schedule

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_device_bytes_match_model(cfg, monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    monkeypatch.setenv("FMG_F3MAT", "0")  # (the model describes the lean form of the 3D kernels,
    monkeypatch.setenv("FMG_TPBY", "0")   #  without its optional 1 byte per point of ý mantissas
    monkeypatch.setenv("FMG_CHK", "0")    #  and without the optional z-chunk buffer)
    import paper_2511_19036_b200 as P
    c = CONFIGS[cfg]
    s = P.Solver(c["dim"], c["p"], c["levels"], default_schedule(c["dim"], c["p"]))
    m = P.memory_model(c["dim"], c["p"], c["levels"])
    modelled = m["fp64_temporary_bytes"] + m["section_bytes"]
    held = s.device_bytes()
    # the model covers sections and FP64 temporaries; the rest (RHS tables,
    # KC scratch, coarse inverse, norm partials, graph bookkeeping) is small
    assert modelled <= held <= modelled * 1.05 + (8 << 20)

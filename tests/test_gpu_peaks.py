"""Same-run compute-peak probes (csrc/peaks.cu, libgftpeaks.so) that bench.py divides by: they
load, run on the device and land in the physically plausible range for one B200."""
import pytest

pytestmark = pytest.mark.gpu


def test_peak_probes_plausible():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    p = bench.measured_compute_peaks(torch.cuda.current_stream())
    assert 40.0 < p["ffma_tflops"] < 90.0            # 148 SMs x 128 lanes x 2 x ~1.9 GHz = 72
    assert 25.0 < p["ffma_reg_tflops"] <= p["ffma_tflops"] * 1.05
    assert 15.0 < p["dfma_tflops"] < 45.0
    assert 600.0 < p["tf32_tflops"] < 1400.0         # dense tcgen05 kind::tf32 ~1.1 PFLOP/s
    assert 25.0 < p["ffma2_tflops"] < 90.0           # packed fma.rn.f32x2, register operands
    assert p["fp32_tflops"] == max(p["ffma_tflops"], p["ffma2_tflops"])

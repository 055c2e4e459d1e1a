"""tcgen05.mma with the A operand in tensor memory (TS mode): layout check."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from test_gpu_kernels import kmajor_image, run_selftest  # noqa: E402


@pytest.mark.parametrize("n", [16, 96])
def test_umma_a_from_tmem(n):
    rng = np.random.default_rng(5)
    K = 96
    a = rng.standard_normal((128, K)).astype(np.float16)
    b = rng.standard_normal((n, K)).astype(np.float16)
    ref = a.astype(np.float32) @ b.astype(np.float32).T
    # A row-major; the kernel packs consecutive K pairs into 32-bit TMEM columns
    got = run_selftest(np.ascontiguousarray(a).reshape(-1), kmajor_image(b), n, K // 16, (0, 0, 0),
                       (n * 16, 128, 2 * n * 16), 2, 0)
    np.testing.assert_allclose(got, ref, rtol=1e-3, atol=1e-2)

"""The fused-dequant GEMMs pick the CTA-pair kernel above 256 tokens and the single-CTA
kernel below (dqgemm.cu / dqgemm_t.cu).  Every shape of tests/test_gpu_dqgemm.py is run
again with each kernel forced (QFT_DQ_PAIR=1 / 0, read once per process, hence the
subprocess): the pair kernel on ragged few-token inputs (tiles mostly out of bounds) and
the single-CTA kernel on many tokens."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("pair", ["1", "0"])
def test_dequant_gemms_with_each_kernel_forced(cuda, pair):
    env = dict(os.environ, QFT_DQ_PAIR=pair)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_dqgemm.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]

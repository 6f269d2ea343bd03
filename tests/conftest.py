import os
import sys

# The oracle is plain single-threaded numpy: pin BLAS / OpenMP pools to one thread
# before numpy loads.  A multi-threaded OpenBLAS pool in the pytest process was
# seen to deadlock in np.linalg.inv after the multi-process GPU test had run
# (GPU box, many cores).
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long CPU test")

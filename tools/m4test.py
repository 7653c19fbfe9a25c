import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"]); sys.path.insert(0, os.path.join(os.environ["GRAFT_REPO_ROOT"], "tests"))
import oracle
from test_gpu_pool import _k23_pool_run
print("err", _k23_pool_run(oracle.port(), 1, 2))

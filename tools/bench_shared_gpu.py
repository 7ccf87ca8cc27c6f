"""Run bench.py's multi-process paths with every rank on cuda:0 over gloo
(the GPU pool here has one GPU; NCCL refuses duplicate devices).  Functional
check only -- ranks share one GPU, so the numbers are not scaling results."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LOCAL_RANK"] = "0"

import torch.distributed as dist  # noqa: E402

_init = dist.init_process_group


def _gloo(backend=None, **kw):
    kw.pop("device_id", None)
    return _init("gloo", **kw)


dist.init_process_group = _gloo
sys.argv[0] = os.path.join(ROOT, "bench.py")
import bench  # noqa: E402

bench.main()

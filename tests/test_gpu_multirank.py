"""The real multi-rank engine path (so2dr_slab_prepare/connect/run: edge bands
pushed GPU-to-GPU into the neighbour's receive buffer over CUDA IPC, ordered by
device-side flag waits) with 2 and 4 processes sharing one B200 -- the only
multi-GPU-shaped run this single-GPU environment allows. Rank 0 reassembles
the grid and checks it bit-for-bit against the oracle, plus the "no halo byte
crosses PCIe twice" invariant (sum of per-rank H2D == one grid per round)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,extra", [(2, {}), (4, {}),
                                         (2, {"SLAB_DIM": "3", "SLAB_KIND": "star", "SLAB_STB": "2",
                                              "SLAB_KON": "2", "SLAB_N": "5"}),
                                         (2, {"SLAB_DTYPE": "f64", "SLAB_KIND": "star"}),
                                         (2, {"SLAB_STB": "6", "SLAB_KON": "4", "SLAB_N": "13"})])
def test_slab_engine_shared_device(world, extra):
    env = dict(os.environ, SO2DR_SHARE_DEVICE="1", **extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tools", "slab_check.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0
    assert "diffs=0 htod_ok=True" in p.stdout

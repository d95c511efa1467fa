"""F2 peer mode across PROCESSES (CUDA IPC, orcha_comm_create_ipc /
ipc_export / ipc_attach): R processes, every one on GPU 0 (the only GPU
here; on a node each would own a GPU and the same mappings go over NVLink),
each mapping the others' packet state, dt gather buffer and barrier counter.
Their result must be bitwise the single-domain run (production build) and
the oracle (parity build), with the same dt / argmax every step on every
rank.  SURVEY 8(f) F2."""
import os
import pickle
import socket
import subprocess
import sys

import numpy as np
import pytest

import orcha_inputs as inp
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import ipc_worker  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(tmp_path, case, mode, steps, method="telescoped"):
    nranks = int(np.prod(ipc_worker.CASES[case][3]))
    out = str(tmp_path / f"ipc_{case}_{mode}_{method}.pkl")
    env = dict(os.environ, ORCHA_PEER_TIMEOUT_MS="60000", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "ipc_worker.py"), out, mode, str(steps), case, method]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    return pickle.load(open(out, "rb"))


def _assemble(g, allr):
    out = None
    for ids, res, _ in allr:
        out = inp.from_blocks(res, g.N, g.nb, ids, out)
    return out


@pytest.mark.parametrize("case", list(ipc_worker.CASES))
def test_ipc_peer_mode_bitwise_equal_single_domain(tmp_path, case):
    nb, nblk, bc, gg, brick, ic = ipc_worker.CASES[case]
    g = H.make_grid(3, nb, nblk, bc=bc)
    U0 = inp.sedov(g.N) if ic == "sedov" else inp.random_field(g.N, seed=91)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=4)
    allr = _run_ranks(tmp_path, case, "production", 4)
    for _, _, log in allr:
        assert log == [tuple(x) for x in logA]
    assert np.array_equal(_assemble(g, allr), A)


def test_ipc_peer_mode_per_stage_variant(tmp_path):
    # F1 + F2 across processes: U1 rows read from other processes' stage-1 buffers
    nb, nblk, bc, gg, brick, ic = ipc_worker.CASES["random16"]
    g = H.make_grid(3, nb, nblk, bc=bc)
    U0 = inp.random_field(g.N, seed=91)
    A, _, logA, _ = H.gpu_run(g, U0, nsteps=3, method="per-stage")
    allr = _run_ranks(tmp_path, "random16", "production", 3, method="per-stage")
    for _, _, log in allr:
        assert log == [tuple(x) for x in logA]
    assert np.array_equal(_assemble(g, allr), A)


def test_ipc_peer_mode_parity_build_equals_oracle(tmp_path):
    nb, nblk, bc, gg, brick, ic = ipc_worker.CASES["sedov8"]
    g = H.make_grid(3, nb, nblk, bc=bc, parity=True)
    U0 = inp.sedov(g.N)
    allr = _run_ranks(tmp_path, "sedov8", "parity", 4)
    Oo, olog = H.oracle_run(H.oracle_grid(g), U0, nsteps=4)
    for _, _, log in allr:
        assert [x[0] for x in log] == olog.dts
        assert [x[2] for x in log] == olog.argmax
    assert np.array_equal(_assemble(g, allr), Oo)


def test_bench_multi_rank_branch_with_ipc_on_one_gpu():
    # bench.py's WORLD_SIZE > 1 branch end to end (torchrun, 2 ranks, F2 peer
    # mode over CUDA IPC, both ranks on GPU 0: ORCHA_BENCH_SAME_GPU=1): one
    # JSON line from rank 0 with the 2-rank workload and per-rank timings
    import json
    env = dict(os.environ, ORCHA_BENCH_SAME_GPU="1", ORCHA_PEER_TIMEOUT_MS="60000", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--comm", "ipc", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-extras"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["comm"] == "ipc" and d["config"]["gpu_grid"] == [2, 1, 1]
    assert d["value"] > 0 and d["nonphysical_first_cell"] == -1

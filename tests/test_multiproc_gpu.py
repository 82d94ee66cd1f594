"""Multi-process paths on one GPU (every rank on device 0): the CUDA-IPC halo
push ring must be bit-identical to a single slab, and bench.py's N>1 code
path must produce its JSON line. Each launch runs under a hard timeout."""
import json
import os
import signal
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def torchrun(nproc, port, *args, timeout=180, env=None):
    """Run in its own process group; on timeout the whole group (launcher and
    every rank) is killed so no rank is left holding the GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", str(nproc), "--master-addr", "127.0.0.1",
           "--master-port", str(port), *map(str, args)]
    p = subprocess.Popen(cmd, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                         text=True, start_new_session=True,
                         env=None if env is None else {**os.environ, **env})
    try:
        out, err = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        out, err = p.communicate()
        pytest.fail(f"{cmd} timed out after {timeout} s\n{out[-2000:]}\n{err[-2000:]}")
    return subprocess.CompletedProcess(cmd, p.returncode, out, err)


@pytest.mark.parametrize("world,scheme", [(2, (2, 1, 1)), (3, (2, 1, 1)), (2, (3, 1, 0)),
                                          (3, (2, 0, 0))])
def test_ipc_ring_processes_bit_identical(world, scheme):
    port = 29610 + 10 * world + scheme[0] + 2 * scheme[2]
    r = torchrun(world, port, "tests/mp/ipc_ring.py", *scheme)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "bit-identical" in r.stdout


@pytest.mark.parametrize("world,scheme", [(2, (2, 1, 1)), (3, (2, 0, 0)), (2, (3, 1, 0))])
def test_ipc_ring_uploaded_fields_bit_identical(world, scheme):
    # uploads of u, v, w, h on an IPC ring must take their static
    # halos from the neighbours (pulled in the first ipc step), not from a
    # self-periodic copy of the rank's own slab.
    port = 29680 + 10 * world + scheme[0] + 2 * scheme[2]
    r = torchrun(world, port, "tests/mp/ipc_ring.py", *scheme, env={"IPC_RING_UPLOAD": "1"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "bit-identical" in r.stdout


def test_bench_two_ranks_json_line():
    r = torchrun(2, 29620, "bench.py", "--gpus", 2, "--one-device", "--config", "c2",
                 "--steps", 3, "--warmup", 3, "--e2e-steps", 1, "--no-cpu-baseline")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["parallelism"] == "slab2 ipc-halo"
    assert line["e2e"]["value"] > 0


def test_bench_gpus_flag_spawns_ranks():
    # `bench.py --gpus N` outside torchrun must launch N
    # ranks itself (one process per GPU) and report n_gpus = N.
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--one-device", "--config", "c2",
           "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline"]
    p = subprocess.Popen(cmd, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                         text=True, start_new_session=True)
    try:
        out, err = p.communicate(timeout=180)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        out, err = p.communicate()
        pytest.fail(f"bench --gpus 2 timed out\n{out[-2000:]}\n{err[-2000:]}")
    assert p.returncode == 0, out[-2000:] + err[-2000:]
    line = json.loads(out.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and len(line["config"]["ranks"]) == 2
    assert {r["rank"] for r in line["config"]["ranks"]} == {0, 1}
    assert "halo path" in err


def test_bench_fpm_shares_from_speed_function():
    # --shares <speed-function CSV>: Algorithm 1 over the ranks (an even split
    # here: the measured B200 speed function satisfies Eq. (1)).
    model = ROOT / "profiles" / "r01_cli_c4" / "speed_avg.csv"
    r = torchrun(2, 29621, "bench.py", "--gpus", 2, "--one-device", "--config", "c2",
                 "--shares", model, "--steps", 3, "--warmup", 3, "--e2e-steps", 1,
                 "--no-cpu-baseline")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["config"]["shares"] == [128, 128]

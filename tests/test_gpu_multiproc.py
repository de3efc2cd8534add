"""The P > 1 path in separate processes (torchrun, one process per rank): CUDA IPC shard mappings, cross-process
device barriers, owner-side gradient collection -- checked against the oracle's union step (reading c.13). With one GPU
the ranks share cuda:0 (same protocol, time-sliced contexts); on a multi-GPU box each rank takes its own device."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(model, P, steps, tmp_path, lag=0, extra=""):
    out = str(tmp_path / f"mp_{model}_{P}_{lag}_{extra}.json")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "mp_dist_worker.py"),
           model, str(steps), out, str(lag), extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return json.load(open(out))


@pytest.mark.parametrize("model", ["transe_l2", "distmult"])
def test_two_processes_match_union_step(model, tmp_path):
    rep = _run(model, 2, 12, tmp_path)
    assert rep["loss_rel"] <= 1e-5, rep
    assert rep["rows"] <= 1e-4 and rep["rel"] <= 1e-4 and rep["states"] <= 1e-5, rep


@pytest.mark.parametrize("lag,extra", [(1, ""), (0, "repartition"), (0, "placement")])
def test_two_processes_variants(lag, extra, tmp_path):
    # separate processes: the lag-1 owner update on the update stream (second barrier sequence), the per-epoch
    # repartition's relation pull over IPC-mapped relation tables (tiny graph at B = 128, P = 2: epochs of 40 steps),
    # head-owner placement with local negatives
    rep = _run("transe_l2", 2, 60 if extra == "repartition" else 12, tmp_path, lag=lag, extra=extra)
    assert rep["loss_rel"] <= 1e-5, rep
    assert rep["rows"] <= 1e-4 and rep["rel"] <= 1e-4 and rep["states"] <= 1e-5, rep

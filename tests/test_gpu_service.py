"""The service loop end to end on the GPU: REQ lines over stdio and over a unix
socket -> ACK, then DONE with logits computed by the B200 manager, checked
against the CPU oracle."""

import io
import socket
import threading
from pathlib import Path

import numpy as np
import pytest

from oracle.executor_ref import run_faithful
from paper_2410_21120_b200 import costmodel, model_io
from paper_2410_21120_b200.repo import Repository
from paper_2410_21120_b200.service import ServiceLoop

pytestmark = pytest.mark.gpu
MODELS = Path(__file__).parent / "golden" / "models"


def make(tmp_path):
    r = Repository(tmp_path / "repo", costmodel.DEFAULT_COST_TABLE)
    for i in range(3):
        r.register_model(model_io.load_graph(MODELS / f"mlp_m{i}.graph.json"),
                         model_io.load_weights(MODELS / f"mlp_m{i}.weights.fiwt"), profile=(50 + 10 * i, 2.0))
    return r, ServiceLoop(r, costmodel.DEFAULT_COST_TABLE, 24_000.0, 10, tmp_path / "out")


def check_done(repo, lines, reqs):
    acks = [l for l in lines if l.startswith("ACK")]
    dones = {l.split()[1]: l.split()[2] for l in lines if l.startswith("DONE")}
    assert len(acks) == len(reqs) == len(dones)
    for (mid, seed), ack in zip(reqs, acks):
        rid = ack.split()[1]
        assert lines.index(ack) < lines.index(next(l for l in lines if l.startswith(f"DONE {rid}")))
        dims, vals = model_io.load_tensor_json(dones[rid])
        g, w = repo.load_pair(mid)
        x = np.random.default_rng(seed).standard_normal(g.input_spec.element_count).astype(np.float32)
        ref = run_faithful(g, w, x)
        assert np.abs(vals - ref).max() <= 2e-2 * max(np.abs(ref).max(), 1e-6)


def test_stdio(tmp_path):
    repo, s = make(tmp_path)
    reqs = [("m0", 3), ("m1", 4), ("m2", 5), ("m0", 6)]
    out = io.StringIO()
    s.serve_stdin(io.StringIO("".join(f"REQ {m} 25 short rand:{k}\n" for m, k in reqs)), out)
    check_done(repo, out.getvalue().splitlines(), reqs)
    assert s.run_logs and all(c.iterate_ms > 0 for lg in s.run_logs for c in lg.cycles)


def test_socket(tmp_path):
    repo, s = make(tmp_path)
    path = tmp_path / "svc.sock"
    ready = threading.Event()
    t = threading.Thread(target=s.serve_socket, args=(path, ready), daemon=True)
    t.start()
    assert ready.wait(30)
    reqs = [("m1", 8), ("m2", 9)]
    c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    c.connect(str(path))
    c.sendall("".join(f"REQ {m} 10 short rand:{k}\n" for m, k in reqs).encode())
    c.shutdown(socket.SHUT_WR)
    data = b""
    while True:
        chunk = c.recv(4096)
        if not chunk:
            break
        data += chunk
    c.close()
    s.stop()
    t.join(60)
    check_done(repo, data.decode().splitlines(), reqs)

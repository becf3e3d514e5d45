"""Service protocol (paper_2410_21120_b200/service.py), host side: parsing and the
immediate ACK / REJ / ERR replies of the reference's ServiceLoop
(service.py:66-104); no execution lane is started."""

from pathlib import Path

from paper_2410_21120_b200 import costmodel, model_io
from paper_2410_21120_b200.repo import Repository
from paper_2410_21120_b200.service import ServiceLoop

MODELS = Path(__file__).parent / "golden" / "models"


def loop(tmp_path):
    r = Repository(tmp_path / "repo", costmodel.DEFAULT_COST_TABLE)
    for i in range(2):
        r.register_model(model_io.load_graph(MODELS / f"mlp_m{i}.graph.json"),
                         model_io.load_weights(MODELS / f"mlp_m{i}.weights.fiwt"), profile=(50 + 10 * i, 2.0))
    return ServiceLoop(r, costmodel.DEFAULT_COST_TABLE, 24_000.0, 10, tmp_path / "out")


def test_replies(tmp_path):
    s = loop(tmp_path)
    got = []
    assert s.handle_line("REQ m0 5 short zeros", got.append) == "req00001"
    assert s.handle_line("REQ ghost 5 short zeros", got.append) is None
    assert s.handle_line("REQ m1 0 short zeros", got.append) is None
    assert s.handle_line("REQ m1 x short zeros", got.append) is None
    assert s.handle_line("HELLO", got.append) is None
    assert s.handle_line("   ", got.append) is None
    assert s.handle_line("REQ m1 3 long rand:7", got.append) == "req00004"
    assert got == ["ACK req00001", "REJ unknown-model", "REJ iterations-must-be->=-1", "ERR parse", "ERR parse",
                   "ACK req00004"]
    assert [r.request_id for r in s.queue.snapshot()] == ["req00001", "req00004"]

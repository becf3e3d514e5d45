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


def test_parse_request_grammar():
    import pytest
    from paper_2410_21120_b200.service import ParseError, Request, parse_request
    assert parse_request("REQ m0 5 short zeros") == Request("m0", 5, "short", "zeros")
    assert parse_request("  REQ m0 -1 long rand:3 \n") == Request("m0", -1, "long", "rand:3")
    assert parse_request("") is None and parse_request(" \t\n") is None
    for bad in ("REQ m0 5 short", "REQ m0 5 short zeros extra", "ACK x", "REQ m0 five short zeros",
                "req m0 5 short zeros"):
        with pytest.raises(ParseError):
            parse_request(bad)


def test_stdio_transport_replies_without_gpu(tmp_path):
    """serve_stdin with requests that are all refused at ingest: the lane never
    needs the GPU, every line is answered in order and EOF returns."""
    import io
    s = loop(tmp_path)
    out = io.StringIO()
    s.serve_stdin(io.StringIO("REQ ghost 5 short zeros\nbad line\n\nREQ m1 0 short zeros\n"), out)
    assert out.getvalue().splitlines() == ["REJ unknown-model", "ERR parse", "REJ iterations-must-be->=-1"]

"""Row f2: the additive `tiler` statement (host logic; the reference parser is used where present)."""

import sys
from pathlib import Path

import pytest

from oracle import aol_oracle as orc
from paper_1105_4424_b200 import Tiler, build_schedule, check_task_signature
from paper_1105_4424_b200.tiler_dsl import TilerSyntaxError, extract_tilers, format_tiler, tilers_by_task

REF_SRC = Path("/root/reference/pkg/src")

MATMUL_MODEL = """\
platform p {
  component Host {
    processor cpu : hwProcessor
    memory ram : hwMemory role=hostRam
  }
  component Cu : hwProcessor {
    processor pe : hwProcessor shaped [8]
  }
  component Dev {
    processor cu : Cu shaped [4]
    memory gmem : hwMemory role=deviceGlobal
  }
  component p {
    part host : Host
    part dev : Dev
  }
}
application m {
  component MatMul {
    port a in float32 [64,32]
    port b in float32 [32,48]
    port c out float32 [64,48]
    repeat [64,48]
    deploy matmul
    tiler a origin [0,0] paving [[1,0],[0,0]] fitting [[0],[1]] pattern [32]
    tiler b origin [0,0] paving [[0,0],[0,1]] fitting [[1],[0]] pattern [32]
    tiler c origin [0,0] paving [[1,0],[0,1]] fitting [[0],[0]] pattern [1]
  }
  component m {
    port pa in float32 [64,32]
    port pb in float32 [32,48]
    port pc out float32 [64,48]
    part mm : MatMul
    connect pa -> mm.a
    connect pb -> mm.b
    connect mm.c -> pc
  }
}
allocate data pa onto dev.gmem
allocate data pb onto dev.gmem
allocate data mm.c onto dev.gmem
allocate task mm onto dev.cu
"""


def test_extract_and_format_roundtrip():
    text, tl = extract_tilers(MATMUL_MODEL)
    assert "tiler" not in text and set(tl) == {"MatMul"} and set(tl["MatMul"]) == {"a", "b", "c"}
    g = orc.gemm_tilers(64, 48, 32)
    for port in "abc":
        want = Tiler(g[port]["origin"], g[port]["paving"], g[port]["fitting"], g[port]["pattern"])
        assert tl["MatMul"][port] == want
        line = format_tiler(port, want)
        _, again = extract_tilers(f"component X {{\n{line}\n}}\n")
        assert again["X"][port] == want
    assert extract_tilers("component Y {\n  tiler x origin [-1] paving [[-2]] fitting [[1]] pattern [3]\n}\n")[1][
        "Y"]["x"].origin == (-1,)


def test_malformed_statements():
    with pytest.raises(TilerSyntaxError):
        extract_tilers("component X {\n  tiler a origin [0] paving [[1]] pattern [2]\n}\n")
    with pytest.raises(TilerSyntaxError):
        extract_tilers("tiler a origin [0] paving [[1]] fitting [[1]] pattern [2]\n")
    with pytest.raises(TilerSyntaxError, match="second tiler"):
        extract_tilers("component X {\n" + format_tiler("a", Tiler.identity()) + "\n"
                       + format_tiler("a", Tiler.identity()) + "\n}\n")


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference front-end not present (GPU box)")
def test_reference_parser_accepts_the_rest(monkeypatch):
    sys.dont_write_bytecode = True
    monkeypatch.syspath_prepend(str(REF_SRC))
    import gmodelc
    text, tl = extract_tilers(MATMUL_MODEL)
    model = gmodelc.parse_model(text)
    assert gmodelc.validate_conformance(model) == []
    per_task = tilers_by_task(model, tl)
    assert set(per_task) == {"mm"}
    comp = model.application_components["MatMul"]
    assert check_task_signature("mm", comp, per_task["mm"]).name == "matmul"
    assert build_schedule(model, 3).steps[0].launches[2].range.count == 64 * 48 // 3
    # no tiler lines: the bundled model text (and so its digest) is untouched
    cg = gmodelc.bundled_model_text()
    assert extract_tilers(cg) == (cg, {})

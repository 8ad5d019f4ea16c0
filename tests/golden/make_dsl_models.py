"""Parse tests/golden/dsl/*.gmodel with the UNMODIFIED reference front-end and commit the models.

Run in the build container only (the reference parser is not on the GPU box):

    python tests/golden/make_dsl_models.py

Each .gmodel carries additive ``tiler`` lines (paper_1105_4424_b200/tiler_dsl.py).  They are
stripped by ``extract_tilers``; the remaining text goes through ``gmodelc.parse_model``
(/root/reference/pkg/src/gmodelc/dsl.py:536-571) and ``gmodelc.validate_conformance``; the
parsed Model is stored as plain data (``model_to_dict``) in dsl_models.json next to the
sha256 of the stripped text, so the GPU test can prove the fixture belongs to the text it
re-reads and re-extracts the tilers from.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF_SRC = Path(os.environ.get("GMODELC_SRC", "/root/reference/pkg/src"))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(HERE.parent.parent))

import gmodelc                                                     # noqa: E402

from paper_1105_4424_b200.model import model_to_dict               # noqa: E402
from paper_1105_4424_b200.tiler_dsl import extract_tilers         # noqa: E402


def main() -> None:
    out = {}
    for path in sorted((HERE / "dsl").glob("*.gmodel")):
        stripped, tilers = extract_tilers(path.read_text())
        model = gmodelc.parse_model(stripped)
        problems = gmodelc.validate_conformance(model)
        assert problems == [], (path.name, problems)
        out[path.stem] = {"sha256": hashlib.sha256(stripped.encode()).hexdigest(),
                          "model": model_to_dict(model),
                          "tiler_components": sorted(tilers)}
    (HERE / "dsl_models.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(out)} models")


if __name__ == "__main__":
    main()

"""Compiles a document that declares a `transmission_line` (lines.expand_document ->
the reference compiler -> lines.bergeron_batch) into tests/golden/lines/line_doc.*,
so the GPU test can run it on the box (no /root/reference there).

    make -C oracle ref && python tools/make_line_doc_fixture.py
"""
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import ref  # noqa: E402
from paper_1903_01081_b200 import lines  # noqa: E402
from paper_1903_01081_b200 import schedule as sch  # noqa: E402
import test_line_document as tl  # noqa: E402

out = os.path.join(ROOT, "tests", "golden", "lines")
doc = tl.line_doc(tau=6.6 * tl.DT, load=250.0)
b = lines.document_batch(doc, tl.reference_compile)
ext = b.initial.size // b.width
with gzip.open(os.path.join(out, "line_doc.cgmsched.gz"), "wt", compresslevel=9) as f:
    f.write(b.text())
with gzip.open(os.path.join(out, "line_doc.state.gz"), "wt", compresslevel=9) as f:
    f.write(sch.format_state(b.initial, ext, b.width))
with open(os.path.join(out, "line_doc.document.json"), "w") as f:
    f.write(json.dumps(json.loads(doc), indent=1) + "\n")
print("line_doc:", b.text().splitlines()[1])

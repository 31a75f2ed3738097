#!/usr/bin/env python3
"""Print the structural fingerprints of the reference corpus functions.

fingerprint = sha256(to_sexpr(fn.params) + "|" + to_sexpr(fn.body)), where
to_sexpr is the reference's own structural dump (trident/syntax.py:303-320:
spans and sem_* annotations excluded, so formatting and comments do not
matter).  The function NAME is excluded on purpose.  The output is pasted
into paper_2305_03317_b200/corpus.py; tests/test_host.py re-derives it when
the reference is importable.
"""
import hashlib
import os
import sys

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
from trident.parser import parse_source  # noqa: E402
from trident.sema import analyze  # noqa: E402
from trident.syntax import to_sexpr  # noqa: E402


def fingerprint(fn):
    s = to_sexpr(fn.params) + "|" + to_sexpr(fn.body)
    return hashlib.sha256(s.encode()).hexdigest()


for name in ("sssp", "sssp_pull", "pr", "bc", "tc", "reduction"):
    p = os.path.join(REF, "trident", "corpus", "programs", name + ".sp")
    tp = analyze(parse_source(open(p).read()))
    print(f'    "{name}": "{fingerprint(tp.function())}",')

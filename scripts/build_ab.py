#!/usr/bin/env python
"""Build A/B variants of libspuma with extra -D defines into build/ab_<tag>.so (loaded by setting
SPUMA_LIBRARY).  usage: python scripts/build_ab.py tag DEFINE=VAL [DEFINE=VAL ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_22215_b200 import _build  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
print(_build.build(defines=defs, out=os.path.join(ROOT, "build", f"ab_{tag}.so")))

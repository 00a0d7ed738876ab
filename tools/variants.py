"""Build tuning variants of librba.so (compile-time pipeline parameters) next to the product
library, for A/B timing with tools/time_matvec.py (RBA_LIB=<variant> python tools/time_matvec.py).
Usage: python tools/variants.py NAME DEFINE [DEFINE ...]   e.g.  v4 RBA_SP_STAGES=4 RBA_SP_VCAP=0"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_01843_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
print(_build.build(force=True, defines=defs, out=os.path.join(_build.HERE, f"librba_{name}.so")))

"""Build the RBA_CHECKS variant of librba (device-side bounds checks that trap) next to the product
library: paper_2103_01843_b200/librba_checked.so.  Run the GPU tests against it with
    RBA_LIB=$PWD/paper_2103_01843_b200/librba_checked.so python -m pytest tests -m gpu
(compute-sanitizer is closed on this pool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_01843_b200 import _build  # noqa: E402

print(_build.build(defines=["RBA_CHECKS"], out=os.path.join(_build.HERE, "librba_checked.so")))

"""One backward with the CTA-pair tcgen05 GEMMs, then one with cuBLAS (for paired ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.lmhead_bwd_once import main  # noqa: E402

if __name__ == "__main__":
    main(4096, 8192, 0)
    main(4096, 8192, 1)

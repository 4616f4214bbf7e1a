"""`python -m paper_2203_03341_b200 <command> ...`: the reference CLI's commands
(`tcgemm split-stats | underflow | gemm-accuracy | rounding-ablation |
ablate-delta`, cli.py:227-265) with their GPU implementations (accuracy.py)."""

import sys

from .accuracy import main

if __name__ == "__main__":
    sys.exit(main())

"""``python -m paper_1711_00231_b200``: the benchmark CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())

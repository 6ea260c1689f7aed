"""``python -m paper_2304_12168_b200 ...``: the command line (cli.py)."""

import sys

from .cli import main

sys.exit(main())

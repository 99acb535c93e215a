"""``python -m paper_1606_08905_b200 ...``: the command line (cli.py)."""

import sys

from .cli import main

sys.exit(main())

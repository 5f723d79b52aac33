"""`python -m paper_2403_08084_b200 ...` runs the experiment CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())

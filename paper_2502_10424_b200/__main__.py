"""python -m paper_2502_10424_b200 run | gamma-sweep | ablate | gen-model (see cli.py)."""

import sys

from .cli import main

sys.exit(main())

"""`python -m paper_2106_15740_b200 ...` — see cli.py."""
import sys

from .cli import main

sys.exit(main())

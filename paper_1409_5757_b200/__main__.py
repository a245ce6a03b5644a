"""`python -m paper_1409_5757_b200 ...` runs the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())

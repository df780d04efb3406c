"""``python -m paper_2510_20271_b200`` runs the ``ecc`` command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())

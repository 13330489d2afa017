"""``python -m paper_1903_02153_b200 {evaluate,bench} ...`` (reference cli.py)."""
import sys

from .cli import main

sys.exit(main())

"""python -m paper_1811_01490_b200 <command> ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

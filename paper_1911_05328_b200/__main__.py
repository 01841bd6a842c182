"""python -m paper_1911_05328_b200 {run,bench,verify} -- see cli.py."""
import sys

from .cli import main

sys.exit(main())

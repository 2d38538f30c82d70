"""python -m paper_2503_10855_b200 ...: see cli.py."""
import sys

from .cli import main

sys.exit(main())

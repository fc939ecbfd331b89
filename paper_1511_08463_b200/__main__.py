"""`python -m paper_1511_08463_b200 run|sweep|validate cfg.ini` (reference cli.py)."""
import sys

from .runio import main

sys.exit(main())

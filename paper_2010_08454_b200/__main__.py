"""`python -m paper_2010_08454_b200 run|bench ...` (cli.py)."""
import sys

from .cli import main

sys.exit(main())

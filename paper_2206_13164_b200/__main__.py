"""python -m paper_2206_13164_b200 solve --config FILE ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())

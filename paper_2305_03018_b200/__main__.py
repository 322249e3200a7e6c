"""python -m paper_2305_03018_b200 ...  ->  the ``morph`` command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())

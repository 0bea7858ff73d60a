"""`python -m paper_2311_04362_b200 <subcommand>`: the experiment CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())

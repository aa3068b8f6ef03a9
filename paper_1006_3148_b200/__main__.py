"""`python -m paper_1006_3148_b200 <subcommand>` — see cli.py."""
import sys

from .cli import main

sys.exit(main())

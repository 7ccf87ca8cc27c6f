"""`python -m paper_1804_07250_b200 sample|cftp|density|hist ...` (cli.py)."""

import sys

from .cli import main

sys.exit(main())

"""``python -m paper_2412_05824_b200`` — the CLI (reference __main__.py)."""

import sys

from .cli import main

sys.exit(main())

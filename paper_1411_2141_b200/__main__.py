"""`python -m paper_1411_2141_b200 ...`: the reference's `meshreg` command line."""
import sys

from .cli import main

sys.exit(main())

"""`python -m paper_2505_22631_b200 ...` == the reference's `python -m oscim ...` (oscim/__main__.py:1-6)."""
import sys

from .cli import main

if __name__ == "__main__":
    sys.exit(main())

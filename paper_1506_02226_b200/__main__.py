"""`python -m paper_1506_02226_b200 ...` = the densescan CLI (cli.py)."""

from .cli import entry

entry()

"""`python -m paper_2209_02878_b200 ...`: the reference's `raysurf` CLI
(raysurf/__main__.py, io_cli.py:239-282) on the B200 engine."""

from .io_cli import main

main()

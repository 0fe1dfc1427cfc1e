"""python -m paper_2402_04403_b200 <subcommand> ... (the reference's `gee` console script)."""

from .cli import main

main()

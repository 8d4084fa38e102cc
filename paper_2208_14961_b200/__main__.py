"""``python -m paper_2208_14961_b200`` == the reference's ``hadamard-ga`` entry point (cli.py:293-294)."""

from .cli import run

run()

"""``python -m paper_2404_16990_b200 simulate|validate|bench ...`` (cli.py)."""
import sys

from .cli import main

sys.exit(main())

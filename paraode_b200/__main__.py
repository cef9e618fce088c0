"""python -m paraode_b200 solve|benchmark|compare (cli.py)."""
import sys

from .cli import main

sys.exit(main())

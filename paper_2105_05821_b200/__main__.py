"""python -m paper_2105_05821_b200 simulate ... (the reference CLI's simulate on the GPU)."""
import sys

from .cli import main

sys.exit(main())

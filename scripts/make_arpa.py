"""CLI of the consistent-backoff synthetic ARPA generator
(paper_2506_00185_b200/lmgen.py); the bench / config scripts import it under
this name."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_00185_b200.lmgen import (arpa_successors, make_arpa,  # noqa: E402,F401
                                         make_consistent_arpa)

if __name__ == "__main__":
    import runpy
    runpy.run_module("paper_2506_00185_b200.lmgen", run_name="__main__")

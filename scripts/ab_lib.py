"""A/B helper: run bench.py (or any script) with an alternative build of the
library loaded first (ee.load(path) caches the handle, so the script's own
ee.load() returns it).  Usage: python scripts/ab_lib.py LIB.so script.py [args]"""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_00518_b200 as ee  # noqa: E402

ee.load(os.path.abspath(sys.argv[1]))
script = sys.argv[2]
sys.argv = [script] + sys.argv[3:]
runpy.run_path(script, run_name="__main__")

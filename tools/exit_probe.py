"""Where does a process exit crash? smoke() with faulthandler and markers (GPU box diagnostic)."""
import faulthandler
import os
import sys

faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as g  # noqa: E402
from paper_1605_04809_b200 import nmt  # noqa: E402

g.smoke()
print("after smoke", nmt.device_allocations(), flush=True)
import gc  # noqa: E402
gc.collect()
print("after gc", nmt.device_allocations(), flush=True)

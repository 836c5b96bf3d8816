import os, sys
sys.path.insert(0, ".")
from paper_2605_08524_b200 import native
if len(sys.argv) > 1 and sys.argv[1] != "base":
    native._LIB_PATH = os.path.abspath(f"dbg/libfcpb_{sys.argv[1]}.so")
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open("scripts/debug_bwd.py").read())

"""Re-run one draw of tools/fuzz_parity.py (same generator): python tools/fuzz_one.py SEED"""
import os, sys, runpy
seed = int(sys.argv[1])
sys.argv = ["fuzz_parity.py", "1", str(seed)]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "fuzz_parity.py"), run_name="__main__")

"""Runs bench.c3_straggler_demo once (debug helper)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench
print(bench.c3_straggler_demo(steps=int(sys.argv[1]) if len(sys.argv) > 1 else 3, warmup=2))

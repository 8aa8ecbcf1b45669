"""One K4 launch for ncu: L=201, p=12, class 0, m free bits (default 26)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_07222_b200 as labs  # noqa: E402
m = int(sys.argv[1]) if len(sys.argv) > 1 else 26
hits, st = labs.enumerate_class(201, 12, 0, m, 4040, collect=False)
print(f"m={m} configurations={st['configurations']} kernel_ms={st['kernel_ms']:.3f} "
      f"steps/s={st['configurations'] / st['kernel_ms'] * 1e3:.3e}")

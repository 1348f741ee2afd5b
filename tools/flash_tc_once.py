"""One antkv_prefill_attention call at n tokens (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from flash_tc_check import run  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
print(run(n, 32, 8)[3])

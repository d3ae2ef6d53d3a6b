"""Replay stress cases (tools/stress_parity.py's dicts, one JSON object per line on stdin)
against the oracle with the current library (BOS_LIBRARY / BOS_THREAD_KERNEL honoured)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import stress_parity  # noqa: E402

for line in sys.stdin:
    line = line.strip()
    if not line:
        continue
    k = json.loads(line)
    k.setdefault("variant", "paper")
    k.setdefault("subarray", 3)
    mx, rms, nan, exc = stress_parity.run_case(k)
    print(json.dumps({"M": k["M"], "snr": k["snr"], "H": k["H"], "W": k["W"], "max": mx, "rms": rms, "nan": nan,
                      "kernel": os.environ.get("BOS_THREAD_KERNEL", "auto"),
                      "lib": os.path.basename(os.environ.get("BOS_LIBRARY", "") or "default")}), flush=True)

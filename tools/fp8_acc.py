"""FP8 accuracy probe for one env setting (FA3B_FP8_THR / FA3B_FP8_VHI are read
once per process): median rmse.v1 rows at N = 1024 and 8192 (d 128, outliers)."""
import json, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2407_08608_b200 import report

tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FA3B_"))
for n, trials in ((1024, 4), (8192, 2)):
    s = report.rmse_rows(n, 128, trials, 1, False)
    med = {k: float(np.median(v)) for k, v in s.items()}
    print(json.dumps({"env": tag, "n": n, **{k: round(v, 6) for k, v in med.items()},
                      "ratio_baseline": round(med["fp8-baseline"] / med["fp8-full"], 3)}), flush=True)

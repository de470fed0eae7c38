#!/usr/bin/env python
"""Fit the alpha-beta model of Eq. 13 to All-Scan measurements (scripts/allscan_bench.py output).

    python scripts/calibrate_costmodel.py profiles/r01_allscan_virtual.jsonl > profiles/costmodel_fit.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_01004_b200 import costmodel as cm  # noqa: E402

path = sys.argv[1]
rep = cm.calibration_report(cm.samples_from_bench(open(path)))
rep["source"] = os.path.basename(path)
print(json.dumps(rep, indent=1))

"""Summarise fill_lab JSON lines: python tools/lab/filllab_summary.py file"""
import json
import sys

for line in open(sys.argv[1]):
    try:
        d = json.loads(line)
    except ValueError:
        print(line.rstrip())
        continue
    name = d.pop("lib").split("libshv_")[-1]
    print(f"{name:12s}", "  ".join(f"{k}={v.get('ms_best', v.get('ms'))}" for k, v in d.items()))

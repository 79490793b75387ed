#!/usr/bin/env python
"""Pivot latency JSON lines (tools/latency.py, tools/latency_mp.py) into one row
per (k, P) with a column per flavour (us per exchange)."""
import collections
import json
import sys

for f in sys.argv[1:]:
    t = collections.defaultdict(dict)
    cols = []
    for line in open(f):
        try:
            r = json.loads(line)
        except Exception:
            continue
        us = r.get("us", r.get("us_max_over_ranks"))
        if us is None:
            continue
        name = "direct" if r.get("path") == "direct" else (r.get("flavour") or "default")
        if name == "default":
            name = f"default({r.get('kernel')})"
        if name.startswith("default"):
            t[(r["k"], r["P"])]["default"] = f"{us:.1f} {r.get('kernel')}"
            name = "default"
        else:
            t[(r["k"], r["P"])][name] = f"{us:.1f}"
        if name not in cols:
            cols.append(name)
    print(f"== {f}")
    print("| k | P | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for key in sorted(t):
        print(f"| {key[0]} | {key[1]} | " + " | ".join(t[key].get(c, "") for c in cols) + " |")

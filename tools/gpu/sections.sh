#!/bin/bash
# every bench side section in its own process: which one errors
for s in overhead c3 c3live c1 jct c4 c2b evict sched c3rate online; do
  echo "== $s"; timeout 400 python bench.py --only $s 2>&1 | tail -1 | grep -oE '"error": "[^"]*"|^\{"[a-z0-9_]*": \{"[a-z_]*"' | head -3
done

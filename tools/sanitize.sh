#!/bin/bash
# compute-sanitizer over small forwards of every hot-path kernel (run on the GPU box).
export PYTHONDONTWRITEBYTECODE=1
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python tools/sanitize_probe.py 2>&1 | grep -v "^{'" | tail -8
done

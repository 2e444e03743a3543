#!/bin/bash
# build library variants for tools/ab.sh: tools/ab_build.sh name "-DFLAG=.." [name "-D.." ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
while [ $# -ge 2 ]; do
  n=$1; x=$2; shift 2
  LPSIM_NVCC_EXTRA="$x" python - "$n" <<'PY'
import os, shutil, sys
sys.path.insert(0, "paper_2406_08496_b200")
import build
b = build
b.OUT = os.path.abspath("ab/%s.so" % sys.argv[1])
b.build(force=True)
print(b.OUT)
PY
done

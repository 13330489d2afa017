#!/bin/bash
# One full-size run of the real reference per BASELINE config.
# C4 fits the builder container (62 GB); C3 and C5 need the GPU host's RAM
# (196 GB): run there with the unmodified reference from baseline/_ref, e.g.
#   gpurun -- 'bash scripts/gen_full_fixtures.sh c5full'
# Outputs tests/golden/<config>_full.npz (copied to gpurun_out/ on the box).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
export BOXFMM_SRC="${BOXFMM_SRC:-$ROOT/baseline/_ref}"
[ -d /root/reference/pkg/src/boxfmm ] && export BOXFMM_SRC=/root/reference/pkg/src
mkdir -p "$ROOT/gpurun_out"
for c in "$@"; do
  python "$ROOT/tests/golden/make_golden.py" "$c"
  f="$ROOT/tests/golden/${c%full}_full.npz"
  [ -f "$f" ] && cp "$f" "$ROOT/gpurun_out/" || true
done

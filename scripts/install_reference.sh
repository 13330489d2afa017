#!/bin/bash
# Install the UNMODIFIED reference (boxfmm, pure Python) into baseline/_ref:
# the bench's reference arm / cpu_baseline and the full-size fixture runs on
# the GPU host import it from there (baseline/_ref is git-ignored, not
# gpurun-ignored, so it travels with the snapshot).  /root/reference is
# read-only, so the build runs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
rm -rf /tmp/boxfmm_src
cp -r /root/reference/pkg /tmp/boxfmm_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade /tmp/boxfmm_src
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import boxfmm; print('boxfmm', boxfmm.__file__)"

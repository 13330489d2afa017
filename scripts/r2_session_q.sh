#!/bin/bash
# Round-2 session Q: full gpu suite on the flag-free P2P (incl. tile-kernel own-cell variant), C5/C4 kernel times.
O=gpurun_out/r2q
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in C5 C4; do
  BFMM_PROFILE=1 timeout 600 python scripts/one_config.py $c > $O/${c}_kernels.log 2>&1
done
echo done

#!/bin/bash
# tools/build_variant.sh <name> "<nvcc -D flags>"  ->  paper_2408_11971_b200/_lib/var_<name>.so
cd "$(dirname "$0")/.."
HSZ_B200_LIB=$PWD/paper_2408_11971_b200/_lib/var_$1.so HSZ_NVCC_EXTRA="$2" \
  python -c "from paper_2408_11971_b200 import build as b; print(b.build(force=True))"

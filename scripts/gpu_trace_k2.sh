#!/bin/bash
# build the measurement library with per-CTA stamps and trace small clouds
set -e
mkdir -p gpurun_out
GS_NVCC_EXTRA="-DGS_TRACE=1" python -c "
from paper_2601_16736_b200 import _build
_build.LIB = _build.PKG / 'build' / 'trace.so'
_build.build(force=True)" > gpurun_out/trace_build.log 2>&1
T=paper_2601_16736_b200/build/trace.so
if [ -n "$TRACE_CASES" ]; then
  eval "$TRACE_CASES"
else
python scripts/trace_k2.py --lib $T --rows 100000 --vis 0.0001 "$@"
python scripts/trace_k2.py --lib $T --rows 100000 --vis 0.5 "$@"
python scripts/trace_k2.py --lib $T --rows 400000 --vis 0.5 "$@"
python scripts/trace_k2.py --lib $T --rows 6250000 --vis 0.01 --fused "$@"
fi

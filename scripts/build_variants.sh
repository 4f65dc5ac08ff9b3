#!/bin/bash
# Build libdx variants in-tree for A/B timing (DX_LIB=libdx_<name>.so selects one at run time).
# Usage: bash scripts/build_variants.sh name1 "flags1" name2 "flags2" ...
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  DX_LIB=libdx_$1.so DX_NVCC_EXTRA="$2" python -c "import importlib.util,sys; s=importlib.util.spec_from_file_location('b','paper_2511_15015_b200/build.py'); b=importlib.util.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)" &
  shift 2
done
wait
ls -la paper_2511_15015_b200/libdx_*.so

#!/bin/bash
# Apply integration/reference_ccg_gpu.patch to a scratch copy of the
# reference's CLI / bench sources and type-check the patched translation
# units, with and without the GPU backend (COOPCG_WITH_GPU).  Needs the
# reference tree (this build container); nothing is written into the repo.
#   bash integration/check_patch.sh [/root/reference/proj]
set -euo pipefail
REF=${1:-/root/reference/proj}
HERE=$(cd "$(dirname "$0")" && pwd)
REPO=$(dirname "$HERE")
W=$(mktemp -d)
trap 'rm -rf "$W"' EXIT
mkdir -p "$W/tools" "$W/src"
cp "$REF/tools/coopcg.cpp" "$REF/tools/CMakeLists.txt" "$W/tools/"
cp "$REF/src/bench.cpp" "$W/src/"
cp "$REF/CMakeLists.txt" "$W/"
(cd "$W" && patch -p1 --quiet < "$HERE/reference_ccg_gpu.patch")
INC="-I$HERE/stub -I$REPO/oracle/stub -I$REF/include -I$REPO/include"
for def in "" "-DCOOPCG_WITH_GPU"; do
  for f in tools/coopcg.cpp src/bench.cpp; do
    g++ -std=c++20 -fsyntax-only -fopenmp -Wall -Wextra $def $INC "$W/$f"
    echo "ok ${def:-(cpu build)} $f"
  done
done
grep -q "ccg-gpu" "$W/tools/coopcg.cpp" && grep -q "ccg-gpu" "$W/src/bench.cpp" && echo "patch applied"

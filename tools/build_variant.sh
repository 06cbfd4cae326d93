#!/bin/bash
# Build a copy of the extension with extra nvcc flags into variants/<name>/
# (A/B kernel experiments: TG_ROOT=variants/<name> python tools/nttbench.py).
#   tools/build_variant.sh <name> "<nvcc flags>"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
D="$ROOT/variants/$1"
rm -rf "$D"; mkdir -p "$D"
cp -r "$ROOT/include" "$D/"
mkdir -p "$D/paper_2412_13269_b200"
cp -r "$ROOT/paper_2412_13269_b200/csrc" "$ROOT/paper_2412_13269_b200"/*.py "$D/paper_2412_13269_b200/"
cd "$D" && TG_NVCC_EXTRA="$2" python -c "
import importlib.util
s = importlib.util.spec_from_file_location('b', 'paper_2412_13269_b200/build.py'); m = importlib.util.module_from_spec(s); s.loader.exec_module(m); m.build()"
rm -rf "$D/build"
echo "built variants/$1"

#!/bin/bash
# Copy the package (+ tools, oracle) into scratch_<name>/ and build it there,
# for side-by-side runs of two library variants on one GPU box.  Tooling only.
#   tools/ab_variant.sh <name> [sed-expression-file-for-csrc]
set -e
name=$1
root=$(cd "$(dirname "$0")/.." && pwd)
dst=$root/scratch_$name
rm -rf "$dst" && mkdir -p "$dst"
cp -r "$root/paper_1505_04086_b200" "$root/tools" "$root/oracle" "$root/include" "$dst/"
rm -f "$dst/paper_1505_04086_b200/libgcol_cuda.so"
if [ -n "$2" ]; then python3 "$2" "$dst/paper_1505_04086_b200/csrc"; fi
python3 "$dst/paper_1505_04086_b200/build.py" > /dev/null 2>&1
echo "built $dst"

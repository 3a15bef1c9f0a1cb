#!/bin/bash
# Build libmdsx.so with extra nvcc defines into scratch/libmdsx_<name>.so
#   bash tools/build_variant.sh <name> -DFOO -DBAR=1
set -e
name=$1; shift
tmp=$(mktemp -d)
cp -r /root/repo/paper_2007_11919_b200 /root/repo/include $tmp/
rm -rf $tmp/paper_2007_11919_b200/build $tmp/paper_2007_11919_b200/libmdsx.so
extra=""
for d in "$@"; do extra="$extra \"$d\","; done
sed -i "s|\"--expt-relaxed-constexpr\",|\"--expt-relaxed-constexpr\", $extra|" $tmp/paper_2007_11919_b200/build.py
(cd $tmp && python -c "from paper_2007_11919_b200.build import build_library as b; b()")
mkdir -p /root/repo/scratch
cp $tmp/paper_2007_11919_b200/libmdsx.so /root/repo/scratch/libmdsx_$name.so
rm -rf $tmp
echo built scratch/libmdsx_$name.so

#!/bin/bash
# Build paper_2411_01919_b200/libpmap_<name>.so with extra nvcc flags (A/B
# timing only; the product is libpmap.so): tools/build_variant.sh NAME "-DKNOB=1 ..."
set -e
cd "$(dirname "$0")/.."
name=$1; shift
flags="$*"
out=build/v_$name; mkdir -p $out
objs=""
for f in paper_2411_01919_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
    -Xcompiler -fPIC,-fvisibility=hidden -Iinclude $flags -c -o $out/$b.o $f &
  objs="$objs $out/$b.o"
done
for f in paper_2411_01919_b200/csrc/*.cpp; do
  b=$(basename $f .cpp)
  g++ -O2 -std=c++17 -fPIC -fvisibility=hidden -Iinclude -c -o $out/$b.cpp.o $f
  objs="$objs $out/$b.cpp.o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o paper_2411_01919_b200/libpmap_$name.so $objs
echo built paper_2411_01919_b200/libpmap_$name.so

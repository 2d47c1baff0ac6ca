#!/bin/bash
# Build libsptk.so with extra nvcc flags into $1 (A/B experiments), e.g.
#   tools/ab_build.sh tools/abx/libA.so -DSPTK_ROW_L1='".L1::no_allocate"'
# (tools/abx/ travels to the GPU box with gpurun; tools/ab/ is gpurun-ignored; both git-ignored *.so)
out=$1; shift
tmp=$(mktemp -d)
ncclinc=$(python -c "import paper_1809_09175_b200.build as b; i=b._nccl_device_include(); print(f'-I {i} -DSPTK_NCCL_DEVICE_API=1' if i else '')")
for f in paper_1809_09175_b200/csrc/*.cu; do
  extra=""; [ "$(basename $f)" = comm.cu ] && extra="$ncclinc"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -I include $extra "$@" -c "$f" -o "$tmp/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "$tmp"/*.o -ldl
rm -rf "$tmp"

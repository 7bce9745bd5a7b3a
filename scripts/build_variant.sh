# build a variant of libsketch.so with extra nvcc defines: build_variant.sh OUT.so -DFOO=1 ...
# (F4FLAGS="..." adds flags for sketch_f4.cu only; default "-Xptxas -O1" as in build.py;
#  KFLAGS="..." adds flags for sketch_kernels.cu only)
set -e
OUT="$1"; shift
D=paper_2310_15419_b200/csrc
T=$(mktemp -d)
F4FLAGS="${F4FLAGS--Xptxas -O1}"
for s in sketch_kernels sketch_f4 sketch_jki sketch_api; do
  extra=""; [ "$s" = sketch_f4 ] && extra="$F4FLAGS"; [ "$s" = sketch_kernels ] && extra="$KFLAGS"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" $extra -I include -c $D/$s.cu -o $T/$s.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" $T/*.o -lcudart
rm -rf $T

#!/bin/bash
# build the working tree's csrc/ with extra nvcc flags into paper_2401_16113_b200/libcnpint_$1.so (A/B variants)
NAME=$1; shift
EXTRA="$*"
mkdir -p build/v_$NAME
for f in paper_2401_16113_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O2 \
      --expt-relaxed-constexpr $EXTRA -c $f -o build/v_$NAME/$b.o -Xptxas -v 2> build/v_$NAME/$b.log &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2401_16113_b200/libcnpint_$NAME.so build/v_$NAME/*.o -cudart static

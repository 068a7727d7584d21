#!/bin/bash
# build paper_2401_16113_b200/libcnpint_ab.so from git revision $1 (default HEAD) of csrc/ for same-box A/B runs
REV=${1:-HEAD}
rm -rf /tmp/abtree && mkdir -p /tmp/abtree build/ab
git archive $REV paper_2401_16113_b200/csrc include | tar -x -C /tmp/abtree
for f in /tmp/abtree/paper_2401_16113_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O2 \
      --expt-relaxed-constexpr $EXTRA -I/tmp/abtree/include -c $f -o build/ab/$b.o 2>/dev/null &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2401_16113_b200/libcnpint_ab.so build/ab/*.o -cudart static

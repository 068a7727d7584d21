# Builds the cnpint C-ABI shared library for B200 (sm_100a).  `make` or __graft_entry__.build().
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
FLAGS   := -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr -Xptxas -v
SRC     := $(wildcard paper_2401_16113_b200/csrc/*.cu)
HDR     := $(wildcard paper_2401_16113_b200/csrc/*.cuh paper_2401_16113_b200/csrc/*.h include/*.h)
LIB     := paper_2401_16113_b200/libcnpint.so
OBJ     := $(patsubst paper_2401_16113_b200/csrc/%.cu,build/%.o,$(SRC))

all: $(LIB)

build/%.o: paper_2401_16113_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(ARCH) $(FLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -cudart static

clean:
	rm -rf build $(LIB)

.PHONY: all clean

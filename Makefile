# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2512_24449_b200/csrc/*.cu)
HDR := $(wildcard paper_2512_24449_b200/csrc/*.cuh) include/packkv_b200.h
OBJ := $(patsubst paper_2512_24449_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2512_24449_b200/libpackkv_b200.so

all: $(LIB)

build/%.o: paper_2512_24449_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean

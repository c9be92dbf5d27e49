# Build the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2505_00136_b200/csrc
SRC := $(wildcard paper_2505_00136_b200/csrc/*.cu)
HDR := $(wildcard paper_2505_00136_b200/csrc/*.cuh) $(wildcard paper_2505_00136_b200/csrc/*.h) include/gpb200.h
OBJ := $(patsubst paper_2505_00136_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2505_00136_b200/libgpb200.so

all: $(LIB)

build/%.o: paper_2505_00136_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean

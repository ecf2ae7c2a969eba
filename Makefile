# Builds libhmc.so in-tree for B200 (sm_100a).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same command.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := paper_2507_14652_b200/csrc/hmc.cu
DEPS := $(wildcard paper_2507_14652_b200/csrc/*.cuh) include/hmc.h
LIB := paper_2507_14652_b200/libhmc.so

$(LIB): $(SRC) $(DEPS)
	$(NVCC) $(FLAGS) -Iinclude -shared -o $@ $(SRC) -lnccl 2> build/ptxas.log || (cat build/ptxas.log; false)

all: $(LIB)
clean:
	rm -f $(LIB)
.PHONY: all clean

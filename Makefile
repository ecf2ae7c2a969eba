# Builds libhmc.so in-tree for B200 (sm_100a).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same command.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
# `make DEV=1`: developer build that reads the engine's tuning / profiling knobs (HMC_TC_*, ...)
# from the environment (include/hmc.h "developer knobs"); the product build ignores them
ifeq ($(DEV),1)
FLAGS += -DHMC_DEV
LIB_OUT := paper_2507_14652_b200/libhmc_dev.so
endif
SRC := paper_2507_14652_b200/csrc/hmc.cu
DEPS := $(wildcard paper_2507_14652_b200/csrc/*.cuh) include/hmc.h
LIB := $(or $(LIB_OUT),paper_2507_14652_b200/libhmc.so)
# link the NCCL that ships with torch (same soname, newer than the system copy) and find it at run time
PYTHON ?= python
NCCL_LIB := $(shell $(PYTHON) -c "import os, nvidia.nccl as m; print(os.path.join(list(m.__path__)[0], 'lib'))" 2>/dev/null)
NCCL_LINK := $(if $(NCCL_LIB),-L$(NCCL_LIB) -Xlinker -rpath=$(NCCL_LIB) -l:libnccl.so.2,-lnccl)

$(LIB): $(SRC) $(DEPS)
	$(NVCC) $(FLAGS) -Iinclude -shared -o $@ $(SRC) $(NCCL_LINK) 2> build/ptxas.log || (cat build/ptxas.log; false)

all: $(LIB)
clean:
	rm -f $(LIB)
.PHONY: all clean

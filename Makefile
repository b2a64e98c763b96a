# Build the product library (sm_100a) and the test-only oracle.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NCCL_DIR  ?= $(shell python -c "import os, nvidia.nccl as n; print(os.path.dirname(n.__file__) if n.__file__ else list(n.__path__)[0])")
NVFLAGS   := $(EXTRA) -O3 -std=c++17 $(ARCH) -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off,-O2 -Xptxas -v \
             -I$(NCCL_DIR)/include
LDFLAGS   := -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib
PKG       := paper_2511_15629_b200
LIB       := $(PKG)/libesdp.so
SRCS      := $(PKG)/csrc/esdp.cu
HDRS      := $(wildcard $(PKG)/csrc/*.cuh) include/esdp.h
ORACLE    := oracle/liboracle.so

all: $(LIB) $(ORACLE)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) $(LDFLAGS) 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; exit 1)

$(ORACLE): oracle/esdp_oracle.c oracle/esdp_oracle.h
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ oracle/esdp_oracle.c -lm

clean:
	rm -f $(LIB) $(ORACLE) $(PKG)/ptxas.log

.PHONY: all clean

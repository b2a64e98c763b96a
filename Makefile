# Build the product library (sm_100a) and the test-only oracle.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off,-O2 -Xptxas -v
PKG       := paper_2511_15629_b200
LIB       := $(PKG)/libesdp.so
SRCS      := $(PKG)/csrc/esdp.cu
HDRS      := $(PKG)/csrc/kernels.cuh include/esdp.h
ORACLE    := oracle/liboracle.so

all: $(LIB) $(ORACLE)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; exit 1)

$(ORACLE): oracle/esdp_oracle.c oracle/esdp_oracle.h
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ oracle/esdp_oracle.c -lm

clean:
	rm -f $(LIB) $(ORACLE) $(PKG)/ptxas.log

.PHONY: all clean

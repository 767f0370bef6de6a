# Builds the product library (libgc.so, sm_100a) and the test oracle (liboracle.so).
# __graft_entry__.build() runs `make`.
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-Wall -Xptxas -v
PKG       := paper_1507_05398_b200
SRC       := $(PKG)/csrc
LIB       := $(PKG)/libgc.so
ORACLE    := oracle/liboracle.so

all: $(LIB) $(ORACLE)

$(SRC)/gc_engine.o: $(SRC)/gc_engine.cu $(SRC)/gc_order.cuh $(SRC)/gc_internal.h include/gc.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(SRC)/gc_engine.ptxas.log || (cat $(SRC)/gc_engine.ptxas.log; false)

$(SRC)/gc_abi.o: $(SRC)/gc_abi.cpp $(SRC)/gc_internal.h include/gc.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC,-Wall -x cu -c $< -o $@

$(SRC)/gc_persistent.o: $(SRC)/gc_persistent.cu $(SRC)/gc_screen.cuh $(SRC)/gc_order.cuh $(SRC)/gc_internal.h include/gc.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(SRC)/gc_persistent.ptxas.log || (cat $(SRC)/gc_persistent.ptxas.log; false)

$(SRC)/gc_pipeline.o: $(SRC)/gc_pipeline.cu $(SRC)/gc_screen.cuh $(SRC)/gc_order.cuh $(SRC)/gc_internal.h include/gc.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(SRC)/gc_pipeline.ptxas.log || (cat $(SRC)/gc_pipeline.ptxas.log; false)

$(SRC)/gc_cw64.o: $(SRC)/gc_cw64.cu $(SRC)/gc_internal.h include/gc.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(SRC)/gc_cw64.ptxas.log || (cat $(SRC)/gc_cw64.ptxas.log; false)

$(SRC)/gc_analysis.o: $(SRC)/gc_analysis.cu $(SRC)/gc_internal.h include/gc.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(SRC)/gc_analysis.ptxas.log || (cat $(SRC)/gc_analysis.ptxas.log; false)

$(LIB): $(SRC)/gc_engine.o $(SRC)/gc_abi.o $(SRC)/gc_persistent.o $(SRC)/gc_pipeline.o $(SRC)/gc_analysis.o $(SRC)/gc_cw64.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl -lpthread

$(ORACLE): oracle/greedy_oracle.c
	gcc -O2 -mpopcnt -Wall -pthread -shared -fPIC -o $@ $<

clean:
	rm -f $(SRC)/*.o $(LIB) $(ORACLE) $(SRC)/*.log

.PHONY: all clean

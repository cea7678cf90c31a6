# Build libbsra.so (sm_100a) and the C oracle. `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -v $(if $(WATCHDOG),-DBSRA_WATCHDOG,) $(if $(EXPERIMENTS),-DBSRA_EXPERIMENTS,)
PKG     := paper_2501_01005_b200
SRC     := $(PKG)/csrc
BUILD   := build
OBJS    := $(BUILD)/engine.o $(BUILD)/scheduler.o $(BUILD)/tc_kernels.o $(BUILD)/dist.o
HDRS    := $(wildcard $(SRC)/*.cuh $(SRC)/*.hpp) include/bsra.h include/bsra_dist.h

all: $(PKG)/libbsra.so oracle/liborc.so

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(BUILD)/scheduler.o: $(SRC)/scheduler.cpp $(SRC)/scheduler.hpp | $(BUILD)
	g++ -O2 -std=c++17 -fPIC -Wall -c $< -o $@

$(BUILD)/dist.o: $(SRC)/dist.cpp include/bsra.h include/bsra_dist.h | $(BUILD)
	g++ -O2 -std=c++17 -fPIC -Wall -I/usr/local/cuda/include -c $< -o $@

$(PKG)/libbsra.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -ldl

oracle/liborc.so: oracle/bsra_oracle.c
	gcc -O2 -fopenmp -fPIC -shared -std=c11 -o $@ $< -lm

clean:
	rm -rf $(BUILD) $(PKG)/libbsra.so oracle/liborc.so

.PHONY: all clean

# Builds the product library in-tree (travels to the GPU box with the snapshot) and
# the test-only oracle libraries (oracle/Makefile).
#   paper_2508_08438_b200/libsafekv_b200.so   C ABI of include/safekv_b200.h (sm_100a)
NVCC     ?= /usr/local/cuda/bin/nvcc
JSON_INC ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2508_08438_b200
SRC      := $(PKG)/csrc
LIB      := $(PKG)/libsafekv_b200.so
BUILD    := build
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
CXXFLAGS := -O2 -std=c++20 -fPIC -Wall -Wextra -I/usr/local/cuda/include -I$(JSON_INC)

OBJS := $(BUILD)/kernels.o $(BUILD)/capi.o $(BUILD)/rules.o $(BUILD)/route.o
GENLIB := workload/libskv_gen.so

all: $(LIB) $(GENLIB) oracle

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/kernels.o: $(SRC)/kernels.cu $(SRC)/hash_scan16.cuh $(SRC)/ctx.hpp include/safekv_b200.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas.log || (cat $(BUILD)/ptxas.log; exit 1)

$(BUILD)/capi.o: $(SRC)/capi.cpp $(SRC)/ctx.hpp $(SRC)/rules.hpp include/safekv_b200.h | $(BUILD)
	g++ $(CXXFLAGS) -c $< -o $@

$(BUILD)/rules.o: $(SRC)/rules.cpp $(SRC)/rules.hpp | $(BUILD)
	g++ $(CXXFLAGS) -c $< -o $@

$(BUILD)/route.o: $(SRC)/route.cpp $(SRC)/route.hpp include/safekv_b200.h | $(BUILD)
	g++ $(CXXFLAGS) -c $< -o $@

# bench / test workload generator (not product code; workload/skv_gen.h)
$(GENLIB): workload/skv_gen.cpp workload/skv_gen.h $(SRC)/route.hpp
	g++ -O2 -std=c++20 -fPIC -shared -Wall -Wextra -pthread -o $@ workload/skv_gen.cpp

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lpthread -ldl -lrt

oracle:
	$(MAKE) -C oracle oracle
	@if [ -d /root/reference/proj/include ]; then $(MAKE) -C oracle ref; fi

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > $(BUILD)/libsafekv_b200.sass

clean:
	rm -rf $(BUILD) $(LIB) $(GENLIB)

.PHONY: all oracle sass clean

# A/B variants of the CUDA library (tools/ab.sh): make variant V=name VFLAGS="-DFOO=1"
variant: $(BUILD)/capi.o $(BUILD)/rules.o $(BUILD)/route.o
	mkdir -p variants/$(V)
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c $(SRC)/kernels.cu -o variants/$(V)/kernels.o 2> variants/$(V)/ptxas.log || (cat variants/$(V)/ptxas.log; exit 1)
	g++ $(CXXFLAGS) $(VFLAGS) -c $(SRC)/capi.cpp -o variants/$(V)/capi.o
	$(NVCC) $(ARCH) -shared -o variants/$(V)/libsafekv_b200.so variants/$(V)/kernels.o variants/$(V)/capi.o $(BUILD)/rules.o $(BUILD)/route.o -lcudart_static -lpthread -ldl -lrt

.PHONY: variant

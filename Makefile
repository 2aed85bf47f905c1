# Build of libseraph.so (sm_100a) and the oracle libraries.
#   make            -> product library + oracle C restatement
#   make ref        -> oracle/_ref from /root/reference sources (checker only)
NVCC ?= /usr/local/cuda/bin/nvcc
CXX := /usr/bin/g++
CUDA_HOME ?= /usr/local/cuda
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_1806_00762_b200
SRC := $(PKG)/csrc
BUILD := build/obj
LIB := $(PKG)/libseraph.so

NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -Iinclude -I$(SRC)
CXXFLAGS := -O3 -std=c++20 -fPIC -Wall -Wextra -Iinclude -I$(SRC) -I$(CUDA_HOME)/include
LDFLAGS := -shared -L$(CUDA_HOME)/lib64 -lcudart -ldl -lpthread -Wl,-rpath,$(CUDA_HOME)/lib64

HDRS := include/seraph.h $(wildcard $(SRC)/*.h)
OBJS := $(BUILD)/kernels.o $(BUILD)/devgraph.o $(BUILD)/engine.o $(BUILD)/engine_graph.o $(BUILD)/engine_stream.o $(BUILD)/engine_blocks.o $(BUILD)/vsched.o $(BUILD)/capi.o $(BUILD)/hostgraph.o $(BUILD)/nccl_dyn.o $(BUILD)/loopback.o $(BUILD)/mt64.o $(BUILD)/stager.o $(BUILD)/group.o

.PHONY: all lib oracle ref clean
all: lib oracle

lib: $(LIB)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/kernels.o: $(SRC)/kernels.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas.log || (cat $(BUILD)/ptxas.log; false)

$(BUILD)/devgraph.o: $(SRC)/devgraph.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_devgraph.log || (cat $(BUILD)/ptxas_devgraph.log; false)

$(BUILD)/%.o: $(SRC)/%.cpp $(HDRS) | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(CXX) -o $@ $(OBJS) $(LDFLAGS)

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean


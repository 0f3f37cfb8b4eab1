# Build of the B200 streaming-GNN engine and its test-side checkers.
#
#   make            -> paper_2309_11071_b200/libstreamgnn.so (product: C ABI + sm_100a kernels)
#                      oracle/liboracle.so (C restatement, test infrastructure)
#                      oracle/_ref/libstreamgnn_ref.so (reference compiled from
#                      /root/reference, when that tree exists; test infrastructure)
#                      tools/libsgnn_datagen.so (synthetic benchmark inputs; harness)
#
# Host C++ is compiled with -ffp-contract=off and the CUDA code with --fmad=false:
# the arithmetic contract is separately rounded mul/add (reference tensor.cpp:41-53).

CXX := /usr/bin/g++
NVCC ?= /usr/local/cuda/bin/nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH := -gencode arch=compute_100a,code=sm_100a

PKG := paper_2309_11071_b200
CSRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/libstreamgnn.so

CXXFLAGS := -std=c++20 -O2 -fPIC -fvisibility=hidden -ffp-contract=off -Wall -Wextra -I$(CUDA_HOME)/include
NVFLAGS := -std=c++17 $(ARCH) -O3 -lineinfo --fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xcompiler -ffp-contract=off -diag-suppress 177 -Wno-deprecated-declarations

HOST_SRCS := tensor_io host_graph model synth stats shard_transport capi
HOST_OBJS := $(addprefix $(OBJ)/,$(addsuffix .o,$(HOST_SRCS)))
DEV_OBJS := $(OBJ)/engine.o
HDRS := $(wildcard $(CSRC)/*.hpp) $(wildcard $(CSRC)/device/*.hpp) $(wildcard $(CSRC)/device/*.cuh) \
        include/streamgnn.h include/streamgnn_b200.h

REF_DIR ?= /root/reference/proj

all: $(LIB) oracle/liboracle.so tools/libsgnn_datagen.so ref

$(OBJ):
	mkdir -p $(OBJ)

$(OBJ)/%.o: $(CSRC)/%.cpp $(HDRS) | $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/engine.o: $(CSRC)/device/engine.cu $(HDRS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(HOST_OBJS) $(DEV_OBJS)
	$(CXX) -shared -o $@ $^ -L$(CUDA_HOME)/lib64 -lcudart_static -lpthread -ldl -lrt -Wl,-Bsymbolic \
	  -Wl,--exclude-libs,ALL

oracle/liboracle.so: oracle/sgnn_oracle.c oracle/sgnn_oracle.h
	$(MAKE) -C oracle

tools/libsgnn_datagen.so: tools/datagen.cpp tools/rmat_gen.hpp
	$(MAKE) -C tools

# The reference is compiled only where its sources exist (this container);
# the GPU box uses the prebuilt oracle/_ref/libstreamgnn_ref.so.
ref:
	@if [ -d $(REF_DIR)/src/core ]; then $(MAKE) -f oracle/ref.mk REF=$(REF_DIR); fi

clean:
	rm -rf build $(LIB) oracle/liboracle.so tools/libsgnn_datagen.so

.PHONY: all ref clean

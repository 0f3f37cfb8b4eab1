# Recipe that compiles the UNMODIFIED reference sources (read-only, under
# /root/reference/proj) into oracle/_ref/libstreamgnn_ref.so, together with our
# own thin harness (oracle/ref_harness.cpp) that exposes the reference's C++
# engine (Engine::process_update_round, baseline::affected_inference) over a C ABI
# for parity fixtures and the CPU baseline.
#
# This is TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and
# bench.py's cpu_baseline / --impl reference legs may load the result.
#
# Flags follow SURVEY.md §7-1: C++20, -O3, no -march=native, and
# -ffp-contract=off so the host never fuses the reference's separately rounded
# mul/add (reference tensor.cpp:41-53) into FMA.
#
# usage: make -f oracle/ref.mk REF=/root/reference/proj

REF ?= /root/reference/proj
OUT := oracle/_ref
OBJ := $(OUT)/obj
CXX := /usr/bin/g++
CXXFLAGS := -std=c++20 -O3 -fPIC -ffp-contract=off -w -I$(REF)/src -I$(REF)/include -Itools

CORE := tensor tensor_io graph model hooks checkpoint baseline engine stats synth
OBJS := $(addprefix $(OBJ)/,$(addsuffix .o,$(CORE))) $(OBJ)/capi.o $(OBJ)/ref_harness.o

all: $(OUT)/libstreamgnn_ref.so $(OUT)/streamgnn_ref_cli

# The reference's own CLI (tools/streamgnn_cli.cpp, unmodified) against the
# reference library; CLI11 (git-ignored vendor/ upstream, absent here) is
# replaced by the subset in oracle/cli11_shim. Used to pin `report` output.
$(OUT)/streamgnn_ref_cli: $(REF)/tools/streamgnn_cli.cpp oracle/cli11_shim/CLI11.hpp $(OUT)/libstreamgnn_ref.so
	$(CXX) $(CXXFLAGS) -Ioracle/cli11_shim -o $@ $< -L$(OUT) -lstreamgnn_ref -Wl,-rpath,'$$ORIGIN'

$(OBJ)/%.o: $(REF)/src/core/%.cpp | $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/capi.o: $(REF)/src/capi/capi.cpp | $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/ref_harness.o: oracle/ref_harness.cpp tools/rmat_gen.hpp | $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libstreamgnn_ref.so: $(OBJS)
	$(CXX) -shared -o $@ $(OBJS) -pthread

$(OBJ):
	mkdir -p $(OBJ)

.PHONY: all

# TEST INFRASTRUCTURE ONLY: compiles the reference library from its own sources where
# they lie under /root/reference (read-only, never copied) with the mini-Eigen /
# mini-doctest shims in oracle/ref_shim, into oracle/_ref/ (git-ignored):
#   _ref/libsftref.so  reference library + ref_bridge.cpp (C ABI for ctypes)
#   _ref/ref_tests     the reference's own doctest suites (proj/tests/test_*.cpp minus
#                      test_cli.cpp, which drives the CLI binary) against that library
#   _ref/acceptance    proj/tests/acceptance.cpp (criteria 1-7; criterion 8 drives the
#                      CLI, replaced by ref_cli_stub.cpp, so it fails by construction)
# Not built: src/cli.cpp (needs the vendored CLI11, absent). Never linked by the product.
REF ?= /root/reference/proj
CXX ?= g++
# the reference build's own flags: CMake Release (-O3 -DNDEBUG), C++20, -Wall -Wextra (proj/CMakeLists.txt)
CXXFLAGS ?= -O3 -DNDEBUG -std=c++20 -fPIC -pthread -Wall -Wextra
HERE := $(dir $(abspath $(lastword $(MAKEFILE_LIST))))
OUT := $(HERE)_ref
INC := -I$(HERE)ref_shim -I$(REF)/include
SRCS := signal engine kernels transforms fourier_fit coeff_io sliding_sum eval
TESTS := test_engine test_transforms test_sliding_sum test_kernels test_signal test_fourier_fit test_eval doctest_main
LIB_OBJS := $(SRCS:%=$(OUT)/obj/src_%.o) $(OUT)/obj/ref_bridge.o
TEST_OBJS := $(TESTS:%=$(OUT)/obj/t_%.o)
SHIM := $(wildcard $(HERE)ref_shim/Eigen/*) $(HERE)ref_shim/doctest.h

all: $(OUT)/libsftref.so $(OUT)/ref_tests $(OUT)/acceptance

$(OUT)/obj/src_%.o: $(REF)/src/%.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(OUT)/obj/ref_bridge.o: $(HERE)ref_bridge.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(OUT)/obj/t_%.o: $(REF)/tests/%.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(OUT)/libsftref.so: $(LIB_OBJS)
	$(CXX) $(CXXFLAGS) -shared -o $@ $^

$(OUT)/ref_tests: $(TEST_OBJS) $(LIB_OBJS)
	$(CXX) $(CXXFLAGS) -o $@ $^

$(OUT)/obj/acceptance.o: $(REF)/tests/acceptance.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(OUT)/obj/ref_cli_stub.o: $(HERE)ref_cli_stub.cpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(OUT)/acceptance: $(OUT)/obj/acceptance.o $(OUT)/obj/ref_cli_stub.o $(LIB_OBJS)
	$(CXX) $(CXXFLAGS) -o $@ $^

clean:
	rm -rf $(OUT)

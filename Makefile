# Builds the in-tree shared library paper_2310_16355_b200/libshardweave_b200.so for sm_100a
# and (optionally) the oracle binaries under oracle/_ref.
NVCC      ?= nvcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
NCCL_DIR  ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
NVCCFLAGS := -std=c++17 -O3 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             --expt-relaxed-constexpr -Iinclude -I$(NCCL_DIR)/include -Xptxas -v
CXXFLAGS  := -std=c++17 -O2 -fPIC -fvisibility=hidden -Iinclude -I/usr/local/cuda/include \
             -I$(NCCL_DIR)/include
SRC_DIR   := paper_2310_16355_b200/csrc
BUILD_DIR := build
LIB       := paper_2310_16355_b200/libshardweave_b200.so

CU_SRCS   := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS  := $(wildcard $(SRC_DIR)/*.cpp)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(BUILD_DIR)/%.cu.o,$(CU_SRCS)) \
             $(patsubst $(SRC_DIR)/%.cpp,$(BUILD_DIR)/%.cpp.o,$(CPP_SRCS))
HDRS      := $(wildcard $(SRC_DIR)/*.h $(SRC_DIR)/*.cuh) include/shardweave_b200.h

all: $(LIB) examples/cpp_train_step

$(BUILD_DIR)/%.cu.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD_DIR)
	$(NVCC) $(NVCCFLAGS) -c $< -o $@ 2> $(BUILD_DIR)/$*.ptxas.log || (cat $(BUILD_DIR)/$*.ptxas.log; exit 1)

$(BUILD_DIR)/%.cpp.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(BUILD_DIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath=$(NCCL_DIR)/lib -lpthread -ldl -lrt

clean:
	rm -rf $(BUILD_DIR) $(LIB)

.PHONY: all clean

examples/cpp_train_step: examples/cpp_train_step.cpp include/shardweave_b200.hpp $(LIB)
	$(CXX) -std=c++17 -O2 -Iinclude $< -o $@ -Lpaper_2310_16355_b200 -lshardweave_b200 \
	    -Wl,-rpath,'$$ORIGIN/../paper_2310_16355_b200'

examples: examples/cpp_train_step
.PHONY: examples

# Experiment builds for same-box A/B timing: make variant NAME=<n> DEFS="-D..." -> variants/libsw_<n>.so
# (load with SW_LIB_PATH=variants/libsw_<n>.so)
variant:
	@mkdir -p build_$(NAME) variants
	$(MAKE) LIB=variants/libsw_$(NAME).so BUILD_DIR=build_$(NAME) NVCCFLAGS="$(NVCCFLAGS) $(DEFS)" \
	    variants/libsw_$(NAME).so
.PHONY: variant

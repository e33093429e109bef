# Build of libsemlab_b200.so (sm_100a kernels + C++ host + C-ABI) — in-tree so it travels
# with gpurun snapshots. `make` builds the product; `make -C oracle` builds the CPU checker.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
CUDA_HOME ?= /usr/local/cuda

PKG := paper_2110_07663_b200
SRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/libsemlab_b200.so

ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC,-fopenmp \
           -I$(SRC) -Iinclude $(EXTRA)
CXXFLAGS := -O3 -std=gnu++17 -fPIC -fopenmp -Wall -Wno-unused-function -I$(SRC) -Iinclude -I$(CUDA_HOME)/include

CU_SRCS := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
HDRS := $(wildcard $(SRC)/*.hpp) $(wildcard $(SRC)/*.cuh) include/semlab_b200.h
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CPP_SRCS))

all: $(LIB)

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fopenmp -L$(CUDA_HOME)/lib64 -lcusolver -lnccl -lgomp

ptxas:  # register / spill report of the kernels
	@for f in $(CU_SRCS); do $(NVCC) $(NVFLAGS) -Xptxas -v -c $$f -o /dev/null 2>&1 | grep -E "Compiling entry|registers|spill" ; done

clean:
	rm -rf build $(LIB)

.PHONY: all clean ptxas

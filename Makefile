# Build of the B200 hot path (sm_100a only) and the test oracles.
#
#   make            -> paper_1502_03391_b200/libjofc_gpu.so (C ABI + kernels)
#                      paper_1502_03391_b200/libjofc.so     (C++ drop-in, namespace jofc)
#                      oracle/libjofc_oracle.so             (test oracle, C restatement)
#   make ref        -> oracle/_ref/libjofc_ref.so           (needs /root/reference)
NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     := /usr/bin/g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_1502_03391_b200
CSRC    := $(PKG)/csrc
NVFLAGS := $(EXTRA) -O3 -std=c++17 $(ARCH) -lineinfo -Iinclude -I$(CSRC) \
           -Xcompiler -fPIC,-fopenmp,-Wall -ccbin $(CXX)
GPU_SRC := $(CSRC)/jofc_capi.cu $(CSRC)/capi_init.cu $(CSRC)/capi_ingest.cu $(CSRC)/capi_peer.cu \
           $(CSRC)/capi_nccl.cu \
           $(CSRC)/jofc_weights.cpp $(CSRC)/host_linalg.cpp $(CSRC)/workloads.cpp $(CSRC)/ingest_io.cpp
GPU_HDR := $(wildcard $(CSRC)/*.cuh $(CSRC)/*.h) include/jofc_gpu.h include/jofc_workloads.h
DROPIN_SRC := $(wildcard $(CSRC)/dropin/*.cpp)
DROPIN_HDR := $(wildcard include/jofc/*.hpp)

all: $(PKG)/libjofc_gpu.so $(PKG)/libjofc.so $(PKG)/libjofc_probe.so oracle build/dropin_parity \
     build/jofc

$(PKG)/libjofc_probe.so: $(CSRC)/probe.cu
	$(NVCC) $(NVFLAGS) -shared -o $@ $<

$(PKG)/libjofc_gpu.so: $(GPU_SRC) $(GPU_HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(GPU_SRC) -lgomp -ldl

# kernel experiments: `make exp EXP=-DJOFC_EXP_...` builds the same C ABI with an
# experimental switch into libjofc_gpu_exp.so (selected with JOFC_GPU_LIB)
exp:
	$(NVCC) $(NVFLAGS) $(EXP) -shared -o $(PKG)/libjofc_gpu_$(or $(EXPNAME),exp).so $(GPU_SRC) -lgomp -ldl

$(PKG)/libjofc.so: $(DROPIN_SRC) $(DROPIN_HDR) $(PKG)/libjofc_gpu.so
	$(CXX) -std=c++20 -O2 -fPIC -shared -Iinclude -I$(CSRC) -o $@ $(DROPIN_SRC) \
	    -L$(PKG) -ljofc_gpu -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle all

# C++ parity suite of the drop-in API (run by tests/test_dropin_cpp.py on a GPU)
build/dropin_parity: tests/cpp/dropin_parity.cpp $(PKG)/libjofc.so oracle/jofc_oracle.c
	@mkdir -p build
	$(MAKE) -C oracle all
	$(CXX) -std=c++20 -O2 -Iinclude -Ioracle -o $@ $< -L$(PKG) -ljofc -ljofc_gpu \
	    -Loracle -ljofc_oracle -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,'$$ORIGIN/../oracle'

# command-line front end (tools/jofc_cli.cpp) on the drop-in API + C ABI
build/jofc: tools/jofc_cli.cpp $(PKG)/libjofc.so $(DROPIN_HDR) include/jofc_gpu.h
	@mkdir -p build
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(PKG) -ljofc -ljofc_gpu \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)'

ref:
	$(MAKE) -C oracle ref

sass: $(PKG)/libjofc_gpu.so
	/usr/local/cuda/bin/cuobjdump -sass $< > build_sass.txt

clean:
	rm -f $(PKG)/*.so
	$(MAKE) -C oracle clean

.PHONY: all oracle ref sass clean exp

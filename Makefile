# Top-level build: the product library (sm_100a CUDA + C-ABI + C++ drop-in)
# and the test-only oracle.  `python -c "import __graft_entry__ as g; g.build()"`
# runs this.  cudart is linked statically and the driver API is resolved at
# run time, so libtw.so loads on GPU-less hosts.

NVCC ?= nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Iinclude -Ipaper_2505_11329_b200/csrc -Xptxas -warn-spills
PKG := paper_2505_11329_b200
LIBDIR := $(PKG)/lib
OBJDIR := build/obj

# Link the SYSTEM libstdc++.so.6 by name: a g++ wrapper whose own -B tree has a
# dangling libstdc++.so symlink silently falls back to libstdc++.a, and a
# static copy next to libtw.so's dynamic one corrupts iostream state (and
# would split exception typeinfo across the drop-in boundary).
STDCXX := -l:libstdc++.so.6

KSRC := $(PKG)/csrc/kernels/tw_launch.cu
HSRC := $(PKG)/csrc/host/tw_capi.cu
MPSRC := $(PKG)/csrc/host/tw_mp.cu
KHDR := $(wildcard $(PKG)/csrc/kernels/*.cuh) $(PKG)/csrc/kernels/tw_launch.h
HHDR := $(PKG)/csrc/host/tw_internal.h include/tw/tw.h
SHIM_SRC := $(wildcard $(PKG)/csrc/host/weavesim_*.cpp)
SHIM_HDR := $(wildcard include/weavesim/*.hpp)

.PHONY: all lib shim weave oracle ref cpptests benchtools clean

all: lib shim weave oracle cpptests benchtools

lib: $(LIBDIR)/libtw.so

$(OBJDIR)/tw_launch.o: $(KSRC) $(KHDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/tw_nvls.o: $(PKG)/csrc/kernels/tw_nvls.cu $(KHDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/tw_capi.o: $(HSRC) $(HHDR) $(KHDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/tw_mp.o: $(MPSRC) $(HHDR) $(KHDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/tw_host_io.o: $(PKG)/csrc/host/tw_host_io.cu $(HHDR) $(KHDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIBDIR)/libtw.so: $(OBJDIR)/tw_launch.o $(OBJDIR)/tw_nvls.o $(OBJDIR)/tw_capi.o $(OBJDIR)/tw_mp.o $(OBJDIR)/tw_host_io.o
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -Xlinker --exclude-libs,ALL

# The drop-in C++ API (namespace weavesim) over the C-ABI.
shim: $(LIBDIR)/libweavesim_b200.so

$(LIBDIR)/libweavesim_b200.so: $(SHIM_SRC) $(SHIM_HDR) $(LIBDIR)/libtw.so
	$(CXX) -std=c++20 -O2 -fPIC -shared -Iinclude -o $@ $(SHIM_SRC) -L$(LIBDIR) -ltw -Wl,-rpath,'$$ORIGIN' -pthread $(STDCXX)

# The weave layer runner (links cuBLAS for the synthetic GEMM load).
weave: $(LIBDIR)/libtw_weave.so

$(LIBDIR)/libtw_weave.so: $(PKG)/csrc/weave/tw_weave.cu include/tw/tw_weave.h include/tw/tw.h include/tw/tw_workload.h \
                          $(LIBDIR)/libtw.so $(LIBDIR)/libweavesim_b200.so
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $< -L$(LIBDIR) -ltw -lweavesim_b200 -lcublas -Xlinker -rpath,'$$ORIGIN' \
	  -Xlinker -rpath,/usr/local/cuda/lib64 -Xlinker --exclude-libs,ALL

# The reference's own test cases compiled against the drop-in library.
cpptests: build/tests/test_dropin

build/tests/test_dropin: tests/cpp/test_dropin.cpp $(SHIM_HDR) $(LIBDIR)/libweavesim_b200.so
	@mkdir -p build/tests
	$(CXX) -std=c++20 -O2 -Iinclude -o $@ $< -L$(LIBDIR) -lweavesim_b200 -ltw -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' $(STDCXX)

# The reference's C++ API timed through the drop-in (bench.py's e2e_dropin_f32).
benchtools: build/bench/dropin_bench

build/bench/dropin_bench: tools/dropin_bench.cpp $(SHIM_HDR) $(LIBDIR)/libweavesim_b200.so
	@mkdir -p build/bench
	$(CXX) -std=c++20 -O2 -Iinclude -o $@ $< -L$(LIBDIR) -lweavesim_b200 -ltw -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' $(STDCXX)

oracle:
	$(MAKE) -C oracle oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

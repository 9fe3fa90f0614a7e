# Builds the three native artefacts in-tree (they travel to the GPU box with the gpurun snapshot):
#   oracle/liboracle.so                           CPU oracle (test infrastructure only)
#   paper_2203_10983_b200/inputs/libbnsgen.so      seeded input generators (setup)
#   paper_2203_10983_b200/libbns.so                the product: C-ABI + sm_100a CUDA kernels + NCCL
#   build/gather_ceiling                           measurement tool: gather ceiling of the SpMM access pattern
PY        ?= python
NVCC      ?= /usr/local/cuda/bin/nvcc
SITE      := $(shell $(PY) -c "import sysconfig; print(sysconfig.get_paths()['purelib'])")
NCCL_DIR  := $(SITE)/nvidia/nccl
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_2203_10983_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cpp)
CHDR      := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/bns.h
OBJDIR    := build

all: oracle/liboracle.so $(PKG)/inputs/libbnsgen.so $(PKG)/libbns.so build/gather_ceiling

# measurement tool (not the product): the SpMM access pattern's gather ceiling (scripts/gather_ceiling.cu)
build/gather_ceiling: scripts/gather_ceiling.cu
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -lineinfo -o $@ $<

oracle/liboracle.so: oracle/bns_oracle.cpp
	g++ -O3 -mavx2 -mfma -std=c++17 -fPIC -shared -o $@ $<

$(PKG)/inputs/libbnsgen.so: $(PKG)/inputs/gen.cpp
	g++ -O3 -std=c++17 -fPIC -shared -fopenmp -o $@ $<

OBJS := $(patsubst $(PKG)/csrc/%,$(OBJDIR)/%.o,$(CSRC))

$(OBJDIR)/%.cu.o: $(PKG)/csrc/%.cu $(CHDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Iinclude -I$(NCCL_DIR)/include -dc -o $@ $< 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/%.cpp.o: $(PKG)/csrc/%.cpp $(CHDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) -O2 -std=c++17 $(CXXDEF) -Wno-deprecated-gpu-targets -Xcompiler -fPIC,-Wall -Iinclude -I$(NCCL_DIR)/include -c -o $@ $<

$(PKG)/libbns.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_DIR)/lib

# A/B variant of the product library with another SpMM segment length (BNS_LIB=... selects it at run time)
kseg%: 
	$(MAKE) OBJDIR=build_kseg$* NVFLAGS="$(NVFLAGS) -DBNS_KSEG=$*" CXXDEF="-DBNS_KSEG=$*" $(PKG)/libbns_kseg$*.so LIBOUT=$(PKG)/libbns_kseg$*.so

$(PKG)/libbns_kseg%.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_DIR)/lib

# generic A/B variant: make variant VAR=name DEFS="-DBNS_X=..." -> $(PKG)/libbns_name.so (BNS_LIB selects it)
variant:
	$(MAKE) OBJDIR=build_$(VAR) NVFLAGS="$(NVFLAGS) $(DEFS)" CXXDEF="$(DEFS)" $(PKG)/libbns_$(VAR).so

$(PKG)/libbns_$(VAR).so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_DIR)/lib

clean:
	rm -rf $(OBJDIR) oracle/liboracle.so $(PKG)/inputs/libbnsgen.so $(PKG)/libbns.so

.PHONY: all clean

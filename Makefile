# Top-level build: the product library (sm_100a) and the test oracles.
#
#   make            -> paper_2112_03592_b200/_lib/libaprgpu.so + oracle/
#   make lib        -> product library only
#   make oracle     -> oracle/liboracle.so (+ oracle/_ref/libaprref.so when
#                      /root/reference is present)

NVCC ?= nvcc
PKG := paper_2112_03592_b200
SRC := $(PKG)/csrc
LIB := $(PKG)/_lib/libaprgpu.so
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Iinclude -Xcompiler -fPIC,-ffp-contract=off,-fvisibility=hidden \
           -Xptxas -v --expt-relaxed-constexpr -diag-suppress 1444,2417
CU_SRCS := $(SRC)/api.cu $(SRC)/index.cu $(SRC)/tree.cu $(SRC)/conv.cu $(SRC)/conv_tile.cu $(SRC)/build.cu $(SRC)/tile.cu $(SRC)/reconstruct.cu $(SRC)/validate.cu $(SRC)/pixels.cu $(SRC)/multi.cu $(SRC)/seqsum.cu
CPP_SRCS := $(SRC)/stencil.cpp $(SRC)/io.cpp
HDRS := $(SRC)/internal.cuh $(SRC)/common.cuh include/aprgpu.h
OBJDIR := build/obj
OBJS := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.o,$(CPP_SRCS))

all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; exit 1)

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) -O3 -std=c++17 -Iinclude -Xcompiler -fPIC,-ffp-contract=off,-fvisibility=hidden,-march=x86-64-v2 -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) -shared $(ARCH) -o $@ $(OBJS) -Xcompiler -fPIC -lpthread

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean

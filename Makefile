# Builds the sm_100a shared library behind include/spcp_b200.h (in-tree, so it
# travels to the GPU box with the repo snapshot) and the oracle recipe.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) $(EXTRA) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr \
           -Xptxas -v,-warn-spills
PKG := paper_1702_02241_b200
SRC := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cuh) include/spcp_b200.h

all: $(PKG)/libspcp_b200.so

$(PKG)/libspcp_b200.so: $(SRC)
	$(NVCC) $(NVFLAGS) -o $@ $(PKG)/csrc/spcp_api.cu 2> $(PKG)/csrc/ptxas.log || (cat $(PKG)/csrc/ptxas.log; exit 1)
	@grep -E "spill|error" $(PKG)/csrc/ptxas.log | grep -v " 0 bytes spill" | head -20 || true

clean:
	rm -f $(PKG)/libspcp_b200.so

.PHONY: all clean

# build libpsp.so variants with compile-time overrides: tools/build_variant.sh NAME "-DX=1 ..."
cd "$(dirname "$0")/.." && mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-O2,-ffp-contract=off -Xptxas -v -shared $2 -I include -o variants/$1.so \
  paper_2311_11833_b200/csrc/psp_host.cpp paper_2311_11833_b200/csrc/psp_plan.cpp \
  paper_2311_11833_b200/csrc/psp_kernels.cu paper_2311_11833_b200/csrc/psp_dense.cu paper_2311_11833_b200/csrc/psp_coopg.cu paper_2311_11833_b200/csrc/psp_dataflow.cu > variants/$1.log 2>&1; echo "$1 rc=$?"

# Build an A/B variant of the library: tools/build_variant.sh NAME [-DMACRO=...]
# (output build_ab/NAME.so, selected at run time with CT_LIBRARY=build_ab/NAME.so)
set -e
name=$1; shift
mkdir -p build_ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -Iinclude "$@" -o build_ab/$name.so paper_2005_11976_b200/csrc/*.cu

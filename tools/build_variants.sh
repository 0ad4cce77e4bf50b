# build libodp.so variants with different tiling macros into variants/
set -e
mkdir -p variants
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr "$@" -o variants/$name.so paper_2204_05520_b200/csrc/odp.cu & }
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  build $name $flags
done
wait
ls variants

# build an A/B variant of the library: bash tools/build_variant.sh <name> <nvcc -D flags...>
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -Xcompiler -fvisibility=default -shared "$@" -o paper_1608_04721_b200/libapbf_gpu_$name.so paper_1608_04721_b200/csrc/apbf_gpu.cu

# Build a compile-time variant of the native library for A/B runs (FDP_LIB_PATH=...):
#   bash tools/build_variant.sh NAME "-DMACRO ..."   ->  paper_2507_01154_b200/_fdp_NAME.so
set -e
name=$1; shift
defs="$*"
cd "$(dirname "$0")/.."
out=paper_2507_01154_b200/_fdp_$name.so
obj=/tmp/fdp_variant_$name; mkdir -p $obj
for s in fdp_tc fdp_group fdp_stream fdp_optim fdp_f64 fdp_ghost fdp_simt fdp_params fdp_capi; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -I include --expt-relaxed-constexpr $defs -c paper_2507_01154_b200/csrc/$s.cu -o $obj/$s.o 2>/dev/null &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $obj/*.o -o $out
echo $out

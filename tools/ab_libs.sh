# Alternate compile-time variants of the native library (tools/build_variant.sh) on single layers:
#   bash tools/ab_libs.sh "B,T,P,D;..." name1 name2 ...   (name "base" = _fdp.so)
shapes=$1; shift
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_2507_01154_b200/_fdp_$v.so; fi
    FDP_LIB_PATH=$lib AB_ROUNDS=2 AB_PATH=${AB_PATH:-two_phase} python tools/ab_layer.py "$shapes" base 2>/dev/null | sed "s/\"variant\": \"base\"/\"variant\": \"$v\", \"rep\": $rep/"
  done
done

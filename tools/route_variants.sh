# timing diagnostics of the routing kernel: build variants that each drop one
# ingredient of the tile phase (parity is void in them), then trace/time each
set -e
cd "$(dirname "$0")/.."
OUT=paper_2605_19893_b200/lib/variants
mkdir -p $OUT
build() {  # name, extra nvcc flags
  local d=$OUT/$1; mkdir -p $d/obj
  for src in attend.cu route.cu compress.cu draft_tree.cu abi.cpp policy.cpp planner.cpp; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
      --expt-relaxed-constexpr -Iinclude -Ipaper_2605_19893_b200/csrc $2 \
      -c paper_2605_19893_b200/csrc/$src -o $d/obj/$src.o
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/libspecsv_b200.so $d/obj/*.o
}
if [ "$1" = "build" ]; then
  for v in ${VARIANTS:-base bconst noexp ks16 ks0 noq}; do
    case $v in
      base) build base "";;
      bconst) build bconst "-DROUTE_DIAG_B_CONST";;
      noexp) build noexp "-DROUTE_DIAG_NO_EXP";;
      ks16) build ks16 "-DROUTE_DIAG_KSTEPS=16";;
      ks0) build ks0 "-DROUTE_DIAG_KSTEPS=0";;
      noq) build noq "-DROUTE_DIAG_NO_Q";;
      twice) build twice "-DROUTE_DIAG_TAIL_TWICE";;
    esac
  done
  exit 0
fi
for v in ${VARIANTS:-base bconst noexp ks16 ks0 noq}; do
  echo "== $v"
  SPECSV_LIB=$OUT/$v/libspecsv_b200.so python tools/trace_route.py 2>&1 | grep -E "staged|computed|tiles done|barrier"
  SPECSV_LIB=$OUT/$v/libspecsv_b200.so python tools/time_route.py 2>&1 | tail -1
done

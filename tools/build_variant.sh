# Same-box A/B builds: tools/build_variant.sh <name> "<nvcc -D flags>" <tu.cu>...
# recompiles the named translation units with the extra flags into
# csrc/build_<name>/ and links paper_2507_16991_b200/libgraphmill_b200_<name>.so
# from them plus the default build's other objects (run `make` first).
set -e
NAME=$1; FLAGS=$2; shift 2
C=paper_2507_16991_b200/csrc
mkdir -p $C/build_$NAME
OBJS=""
for o in $C/build/*.o; do
  b=$(basename $o .o)
  hit=""
  for tu in "$@"; do [ "$(basename $tu .cu)" = "$b" ] && hit=1; done
  if [ -n "$hit" ]; then
    /usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -Iinclude -I$C \
      $FLAGS -c $C/$b.cu -o $C/build_$NAME/$b.o &
    OBJS="$OBJS $C/build_$NAME/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o paper_2507_16991_b200/libgraphmill_b200_$NAME.so $OBJS -ldl
echo built paper_2507_16991_b200/libgraphmill_b200_$NAME.so

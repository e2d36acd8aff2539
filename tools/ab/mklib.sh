# Build one variant of the native library without touching the in-tree one (dev tool).
# usage: tools/ab/mklib.sh NAME FILE=variant.cu [FILE=variant.cu ...]
#   compiles every csrc/*.cu once into /tmp/abobj (cached), recompiles the
#   named translation units (extra nvcc flags for them: ABFLAGS) from the given variant sources, links
#   tools/ab/lib_NAME.so.  On the GPU box run tools/ab/swap.sh.
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
CSRC=$ROOT/paper_2002_00552_b200/csrc
OBJ=/tmp/abobj; mkdir -p $OBJ/$name
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I $ROOT/include -I $CSRC"
for src in $CSRC/*.cu; do
  o=$OBJ/$(basename $src .cu).o
  [ -f $o ] || echo "nvcc $FLAGS -c $src -o $o"
done | xargs -P 16 -I{} sh -c "{}"
objs=""
for src in $CSRC/*.cu; do
  b=$(basename $src .cu); o=$OBJ/$b.o
  for kv in "$@"; do
    tu=${kv%%=*}; var=${kv#*=}
    if [ "$tu" = "$b.cu" ]; then
      o=$OBJ/$name/$b.o
      nvcc $FLAGS $ABFLAGS -c $var -o $o
    fi
  done
  objs="$objs $o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/ab/lib_$name.so $objs
echo built tools/ab/lib_$name.so

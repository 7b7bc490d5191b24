# Build a variant library with extra nvcc flags: bash tools/build_variant.sh NAME "-DHODG_X=1 ..."
# -> tools/variants/NAME/libhodg_b200.so (select at run time with HODG_B200_LIB)
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/tools/variants/$NAME
mkdir -p $OUT
make -s -j8 -C $ROOT/paper_2209_01877_b200/csrc OUT=$OUT EXTRA="$FLAGS" $OUT/libhodg_b200.so

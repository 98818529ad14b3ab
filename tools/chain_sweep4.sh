run() { echo "== $*"; env "${@:3}" timeout 900 python tools/p1_epoch.py $1 $2 2>&1 | grep -E "config|rror" | tail -1 | cut -c90-330; }
for lib in "" "GAPLRA_CUDA_LIB=$PWD/build/variants/libgaplra_noticks.so"; do echo "#### $lib"; run C2 1 $lib; run C3 1 $lib; run C2 20 $lib; run C3 32 $lib; run C5 64 $lib; done

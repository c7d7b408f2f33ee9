# Build an A/B variant of the library: bash tools/build_variant.sh NAME "-DMACRO=VALUE ..."
# -> paper_2509_23043_b200/lib/variants/libtapt_NAME.so (select with TAPT_LIB_PATH)
R=$(cd "$(dirname "$0")/.." && pwd)
make -s -j4 -C "$R/paper_2509_23043_b200/csrc" OUT="$R/paper_2509_23043_b200/lib/variants/libtapt_$1.so" \
    BUILD="$R/paper_2509_23043_b200/csrc/build_$1" EXTRA="$2"

# Build an A/B variant of the library into altbuild/ (travels to the GPU box; objects do not):
#   bash tools/build_alt.sh -DEIK_ROWDFT_SPLIT=0
make -j16 OBJ=altbuild/obj LIB=altbuild/libeikfld_b200.so EXTRA="$*" >/dev/null && echo "altbuild/libeikfld_b200.so: $*"

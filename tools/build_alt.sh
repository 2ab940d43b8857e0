# Build an A/B variant of the library into altbuild/ (travels to the GPU box; objects do not):
#   bash tools/build_alt.sh -DEIK_ROWDFT_SPLIT=0
# The objects are rebuilt every time (make does not track EXTRA), so the
# variant always reflects its flags.
rm -rf altbuild/obj altbuild/libeikfld_b200.so
make -j16 OBJ=altbuild/obj LIB=altbuild/libeikfld_b200.so EXTRA="$*" >/dev/null && echo "altbuild/libeikfld_b200.so: $*"

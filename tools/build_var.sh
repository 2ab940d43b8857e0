# Build a named A/B variant of the library into altv/<name>/ (travels to the GPU box):
#   bash tools/build_var.sh il1 -DEIK_F4K_IL=1
name=$1; shift
rm -rf altv/$name
make -j16 OBJ=altv/$name/obj LIB=altv/$name/libeikfld_b200.so EXTRA="$*" >/dev/null && rm -rf altv/$name/obj.keep && echo "altv/$name: $*"

for v in NOUNROLL ASMSYNC NOPIPE; do echo "== $v"; PSP_LIB=$PWD/tools/gpu/libpsp_$v.so timeout 100 python tools/gpu/lz1.py 8; done

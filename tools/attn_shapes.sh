for v in $1; do FB_LIB_PATH=tools/libfedb200_$v.so python tools/attn_shapes.py | sed "s/^/$v /"; done

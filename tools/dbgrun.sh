W3D_NVCC_EXTRA="-DW3D_DEBUG_TMA" python build.py cuda --force > /dev/null 2>&1
python tools/dbg_tma.py 2>&1 | grep -v "^blk" | tail -5

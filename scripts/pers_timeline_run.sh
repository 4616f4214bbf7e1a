i=0; for v in "$@"; do i=$((i+1)); echo "== variant $v#$i"; TCEC_LIB=exp_libs/libtl_$v.so python scripts/pers_timeline.py 2>&1 | sed -n "/=== timed/,\$p"; done

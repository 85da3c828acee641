for c in C2 C4; do for v in "$@"; do
  echo "== $c $v $(MGAUSS_B200_LIB=paper_2603_00145_b200/_lib/var_$v.so timeout 300 python tools/kbench.py --config $c 2>&1 | tail -1 | cut -c1-100)"
done; done

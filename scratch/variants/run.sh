for v in base cicc2 cicc1 cicc0 ptx0; do echo "== $v"; SEL_LIB=scratch/variants/$v.so python scratch/dbg_pd3.py 2>&1 | grep -c BAD ; done

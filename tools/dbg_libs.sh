for L in "$@"; do echo "== $L"; PYTHONPATH=. DILU_LIB=paper_2503_05130_b200/$L python tools/dbg_c2.py 2>&1 | tail -1; done

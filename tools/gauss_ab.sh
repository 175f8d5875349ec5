for l in abvar/g0.so abvar/gpf.so; do cp $l paper_1402_5938_b200/libsfmg.so; echo "== $l"; python tools/gauss_bench.py; done

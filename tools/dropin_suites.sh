#!/bin/bash
# the reference's own doctest suites (built by dropin/Makefile against the drop-in) + the drop-in's own suite, on one B200
O=gpurun_out/dropin_suites.txt
echo "# the reference's own doctest suites (P:tests/test_*.cpp, unmodified) built by dropin/Makefile against the" > $O
echo "# B200 drop-in (dropin/src + dropin/include/tq/{select,project}.hpp -> libcrystal_b200.so), run on one B200 (r02 kernels)" >> $O
for t in test_hash_join test_project test_radix test_select test_ssb test_tile_engine test_dropin_group; do
  echo "== oracle/_ref/dropin/$t" >> $O
  timeout 900 oracle/_ref/dropin/$t > /tmp/o.txt 2>&1; echo "rc=$?" >> $O
  grep -E "test cases|assertions" /tmp/o.txt >> $O
done

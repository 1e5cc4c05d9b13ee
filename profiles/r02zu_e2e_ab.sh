# c2 end to end (tools/e2e_breakdown.py), same box: .ab/base (fd11f39) vs the working tree
for i in 1 2; do for d in .ab/base .; do
  (cd $d && timeout 600 python tools/e2e_breakdown.py 2>&1 | tail -4 | sed "s|^|$d |")
done; done

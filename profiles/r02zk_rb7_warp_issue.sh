# RB7-like model through tc_layer_kernel, same box: .ab/pre = 4850338 (single-thread MMA issue) vs HEAD (warp-issued)
for d in .ab/pre .; do
  for P in tf32x3 bf16; do (cd $d && timeout 300 python profiles/rb7_prof.py $P | sed "s|^|$d |"); done
done

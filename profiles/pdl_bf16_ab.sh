for i in 1 2; do
for P in bf16 fp8; do
  echo "default $P: $(python profiles/prof_run.py --precision $P --runs 3)"
  echo "pdl-all $P: $(SIMNET_PDL=front,layer,layer_bf16 python profiles/prof_run.py --precision $P --runs 3)"
done; done

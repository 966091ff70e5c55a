# A/B of build variants: bash scripts/gpu_ab_libs.sh "lib1 lib2 ..." "workloads" [reps] [rounds]
LIBS=${1:-libsigattn.so}; WLS=${2:-c3}; REPS=${3:-20}; ROUNDS=${4:-2}
for r in $(seq $ROUNDS); do for lib in $LIBS; do for w in $WLS; do
  echo -n "$lib "; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w $REPS 2>&1 | tail -1
done; done; done

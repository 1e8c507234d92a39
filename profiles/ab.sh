# A/B timing of two builds of libglsim_cuda on the same box (dev helper):
# HEAD build as libglsim_cuda_head.so vs the working-copy build, alternated.
# Extra bench arguments (e.g. --config C3 --windows 2048) pass through.
for i in 1 2; do
  for lib in libglsim_cuda_head.so libglsim_cuda.so; do
    printf "%s " $lib; GLSIM_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))"
  done
done

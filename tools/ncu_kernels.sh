# ncu --set full of selected kernels of one bench step (one GPU; only after
# the same bench command exited 0 without ncu).
#   WL=sort_i32 KREGEX="qs_local" TAG=x ENVV="" bash tools/ncu_kernels.sh
mkdir -p gpurun_out/ncu
env $ENVV timeout ${NCU_TIMEOUT:-900} ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-qs_}" -c ${COUNT:-1} --launch-skip ${SKIP:-0} \
  -o gpurun_out/ncu/${TAG:-x} -f python bench.py --workload ${WL:-sort_i32} --steps 1 --warmup 0 --prof-steps 1 --no-e2e --no-cpu \
  > gpurun_out/ncu/${TAG:-x}.log 2>&1
echo "ncu ${TAG:-x} rc=$?"

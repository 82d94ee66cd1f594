mkdir -p gpurun_out
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
for n in cur norhpf base; do
  if [ $n = cur ]; then L=""; else L="IMB_LIB=$PWD/experiments/libimb_$n.so"; fi
  env $L ncu --set full --clock-control none -k regex:k_fused -s 1 -c 1 -o gpurun_out/cf_$n $P > gpurun_out/ncu_$n.log 2>&1; echo $n=$?
done

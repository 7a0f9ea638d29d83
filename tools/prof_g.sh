tools/ab.sh "ring3:X=1" "ring2:INFT_LIB=exp/lib_sg2.so"
for v in "ring3:X=1" "ring2:INFT_LIB=exp/lib_sg2.so"; do n=${v%%:*}; e=${v#*:}
env $e ncu --set full --import-source on --clock-control none -k regex:k_gather_ring -c 1 -o gpurun_out/g_$n -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/ncu_g_$n.log 2>&1
done

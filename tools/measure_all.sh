#!/bin/bash
# Round measurement batch (run on the GPU box through gpurun):
#   bench.py lines for every BASELINE configuration, the ncu launch list
#   (time + DRAM bytes) of each configuration's product, and one
#   `ncu --set full` capture per repeated-addition kernel.
# Output: gpurun_out/$OUT/
OUT=${OUT:-meas}
D=gpurun_out/$OUT
mkdir -p $D
NCU_M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
python bench.py > $D/bench_cfg5.json 2> $D/bench_cfg5.err
python bench.py --impl reference > $D/bench_ref_cfg5.json 2>> $D/bench_cfg5.err
for c in cfg1 cfg2 cfg4; do
  python bench.py --config $c --cpu-seconds 4 > $D/bench_$c.json 2>> $D/bench_other.err
done
for d1 in 0.1 0.5 1.0; do for mu in 1 4 16; do
  python bench.py --config cfg3 --d1 $d1 --mu $mu --cpu-seconds 4 > $D/bench_cfg3_d${d1}_mu${mu}.json 2>> $D/bench_other.err
done; done
# launch lists (each after the same command exited 0 without ncu)
for spec in "cfg1" "cfg2" "cfg4" "cfg5" "cfg3 --d1 0.1 --mu 1" "cfg3 --d1 0.1 --mu 4" "cfg3 --d1 0.1 --mu 16" "cfg3 --d1 0.5 --mu 1" "cfg3 --d1 0.5 --mu 4" "cfg3 --d1 0.5 --mu 16" "cfg3 --d1 1.0 --mu 1" "cfg3 --d1 1.0 --mu 4" "cfg3 --d1 1.0 --mu 16"; do
  tag=$(echo $spec | sed 's/ --d1 /_d/; s/ --mu /_mu/')
  if python tools/profile_one.py $spec > $D/po_$tag.log 2>&1; then
    ncu --metrics $NCU_M --print-units base --clock-control none --csv --log-file $D/launches_$tag.csv python tools/profile_one.py $spec > /dev/null 2>&1
  fi
done
# full captures of the three repeated-addition kernels (already run above without ncu)
ncu --set full --clock-control none --import-source on -k regex:k_aform -c 1 -f -o $D/prof_aform_cfg3_d0.1_mu4 python tools/profile_one.py cfg3 --d1 0.1 --mu 4 > $D/ncu_aform.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bform -c 1 -f -o $D/prof_bform_cfg5_n4096 python tools/profile_one.py cfg5 --n 4096 > $D/ncu_bform.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bgroup -c 1 -f -o $D/prof_bgroup_cfg3_d1.0_mu1 python tools/profile_one.py cfg3 --d1 1.0 --mu 1 > $D/ncu_bgroup.log 2>&1
echo done > $D/DONE

# Round-2 profile set: launch list of the bench command, ncu --set full of the headline
# kernel inside bench.py, and one ncu --set full capture per other benched kernel.
set -x
NO="--no-e2e --no-cpu-baseline --no-next1 --no-next2 --no-next3 --no-next4 --no-configs"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02p_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r02p_launch.log 2>&1; echo launch rc $?
ncu --set full --clock-control none --import-source on -k regex:clip_compact_packed -s 3 -c 1 -f -o gpurun_out/r02p_headline python bench.py --steps 1 --warmup 3 $NO > gpurun_out/r02p_headline.log 2>&1; echo headline rc $?
ncu -i gpurun_out/r02p_headline.ncu-rep --page raw --csv > gpurun_out/r02p_headline_raw.csv
ncu -i gpurun_out/r02p_headline.ncu-rep --page source --csv --print-source sass > gpurun_out/r02p_headline_src.csv
for spec in "dense2d:--kernel dense --n 100000000:clip_dense" "compact3d:--kernel compact --n 100000000 --dim 3:clip_compact_packed" \
            "homog:--kernel compact --n 100000000 --family homog:clip_compact_packed" \
            "homogndc:--kernel compact --n 100000000 --family homog --ndc 1:clip_compact_packed" \
            "adv2d:--kernel compact --n 10000000 --family adv:clip_compact_packed" \
            "adv2d64:--kernel compact --n 10000000 --family adv --dtype f64:clip_compact_packed" \
            "mix33:--kernel compact --n 100000000 --family mix33:clip_compact_packed"; do
  tag=${spec%%:*}; rest=${spec#*:}; args=${rest%%:*}; k=${rest##*:}
  ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -f -o gpurun_out/r02p_$tag python scripts/kernel_probe.py $args --reps 1 > gpurun_out/r02p_$tag.log 2>&1; echo $tag rc $?
  ncu -i gpurun_out/r02p_$tag.ncu-rep --page raw --csv > gpurun_out/r02p_${tag}_raw.csv
done
for k in tof_range_phi_kernel clip_int_kernel cluster_kernel; do
  ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -f -o gpurun_out/r02p_$k python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --no-next1 > gpurun_out/r02p_$k.log 2>&1; echo $k rc $?
  ncu -i gpurun_out/r02p_$k.ncu-rep --page raw --csv > gpurun_out/r02p_${k}_raw.csv
done
rm -f gpurun_out/r02p_*.ncu-rep

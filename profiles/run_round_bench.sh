#!/bin/bash
# Round measurement batch (run on the GPU box from the repo root):
# bench lines for every workload, the reference arm, the C4 launch list, the
# ncu captures of the dominant kernel and of one (warm) C4 V-cycle, per-level
# costs.  Everything lands in gpurun_out/; copy the summaries to profiles/.
O=gpurun_out
mkdir -p $O
python bench.py > $O/b_c4.json 2> $O/b_c4.err
for w in c3 c2 c5 c1; do python bench.py --workload $w > $O/b_$w.json 2> $O/b_$w.err; done
python bench.py --workload c4 --smoother ms --no-device-setup > $O/b_c4_ms.json 2> $O/b_c4_ms.err
python bench.py --workload c5 --smoother ms --no-device-setup > $O/b_c5_ms.json 2> $O/b_c5_ms.err
python bench.py --impl reference > $O/b_ref_c4.json 2> $O/b_ref_c4.err
python profiles/level_costs.py c4 --json $O/level_costs_c4.json > $O/level_costs_c4.log 2>&1
python profiles/spmv_modes.py c4 > $O/spmv_modes_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline --no-device-setup --no-fast-mode > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pspmv -s 1 -c 1 -f -o $O/pspmv_full \
  python profiles/profile_c4.py spmv > $O/ncu_pspmv.log 2>&1
ncu -i $O/pspmv_full.ncu-rep --page raw --csv > $O/pspmv_raw.csv 2>&1
ncu -i $O/pspmv_full.ncu-rep --page source --csv --print-source cuda,sass > $O/pspmv_src.csv 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv \
  --log-file $O/vc_c4.csv python profiles/profile_c4.py vcycle2 > $O/ncu_vc.log 2>&1
echo done

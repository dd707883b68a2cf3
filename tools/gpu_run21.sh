#!/bin/bash
# L2 evict_last on source records + streaming partial stores: DRAM bytes and timing.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python paper_1707_06551_b200/build.py > /dev/null 2>&1
timeout 600 python tools/profile_step.py --config 5 --no-off > gpurun_out/r24_plain.log 2>&1; echo "plain exit $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct \
  --clock-control none -k regex:k_nbody -c 1 python tools/profile_step.py --config 5 --no-off > gpurun_out/r24_ncu.log 2>&1
echo "ncu exit $?"; grep -E "dram__|gpu__time|lts__" gpurun_out/r24_ncu.log
timeout 900 python bench.py > gpurun_out/r24_bench.json 2> gpurun_out/r24_bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r24_bench.json'));print(d['value'],d['roofline']['fp64_pipe_frac'],d['kernels']['nbody'],d['kernels']['offsurface'])"

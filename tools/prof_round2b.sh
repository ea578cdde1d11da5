# Round-2 profiles, part 2: CGS2 sweeps at c = 40 and the per-config report.
set -e
mkdir -p gpurun_out /tmp/p2
[ -n "$SKIP_CONFIGS" ] || python tools/config_report.py 1 2 3 5 4 > gpurun_out/p2_configs.jsonl 2> gpurun_out/p2_configs.err
python tools/prof_kernels.py cgs sell32 > /dev/null 2>&1
# the bare ArnoldiState extends with classical CGS2 (3 sweeps per step); the
# c = 33..40 steps use the CPW = 8 instantiations: skip those 24, capture the
# first cgs2_step at c = 40 (dot, update+dot, store)
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_tspipe<\(int\)[024], \(int\)8>' -s 24 -c 3 \
    -o /tmp/p2/p2_cgs40 python tools/prof_kernels.py cgs sell32 > gpurun_out/p2_ncu5.log 2>&1
python tools/summarize_ncu.py kernels /tmp/p2/p2_cgs40.ncu-rep gpurun_out/p2_cgs40.md p2_cgs40
python tools/ncu_digest.py /tmp/p2/p2_cgs40.ncu-rep 20 > gpurun_out/p2_cgs40_digest.txt 2>&1 || true

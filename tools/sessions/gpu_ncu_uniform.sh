mkdir -p gpurun_out/u2
for k in ${NCU_KS:-64 200}; do
ONCE_K=$k ncu --set full --import-source on -k regex:sketch_uniform -s 1 -c 1 -o gpurun_out/u2/uni_k$k python tools/uniform_once.py > gpurun_out/u2/ncu_k$k.log 2>&1
done

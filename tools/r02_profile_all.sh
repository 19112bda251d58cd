# usage (under gpurun): tools/r02_profile_all.sh <tag>
# GPU suite, default bench, ncu launch list of a short bench, ncu --set full
# captures of the lattice tile kernel (2048^2), SpMV (2048^2), hypercube term (hc_pair_kernel)
# (dim 22) and CSR Taylor term (2048^2 grid H); each ncu run follows the same
# command exiting 0 without ncu (tools/ncu_capture.sh).
set -u
tag=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_gputests.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
B="python bench.py --steps 2 --warmup 3 --walk-steps 40 --no-extras --no-cpu"
$B > gpurun_out/${tag}_plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/${tag}_ncu_launches.log 2>&1
bash tools/ncu_capture.sh ${tag}_tb lattice_tb 8 -- python tools/time_lattice.py 2048 40
bash tools/ncu_capture.sh ${tag}_spmv spmv_kernel 8 -- python tools/time_spmv.py 2048
bash tools/ncu_capture.sh ${tag}_hc hc_pair 6 -- python tools/run_c4.py 22
bash tools/ncu_capture.sh ${tag}_csr csr_term 6 -- python tools/time_ctqw_csr.py 2048
cuobjdump -sass paper_2406_08186_b200/_lib/libqwb200.so > /tmp/all.sass 2>/dev/null
grep -c "UTMALDG" /tmp/all.sass > gpurun_out/${tag}_sass_counts.txt
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_reference.json 2> gpurun_out/${tag}_reference.err
for op in UTMALDG UBLKCP SYNCS.ARRIVE.TRANS64 SYNCS.PHASECHK LDGSTS DADD DMUL; do echo "$op $(grep -c "$op" /tmp/all.sass)"; done >> gpurun_out/${tag}_sass_counts.txt
grep -m3 -B2 -A2 "UTMALDG" /tmp/all.sass > gpurun_out/${tag}_sass_excerpt.txt
grep -m3 -B2 -A2 "UBLKCP" /tmp/all.sass >> gpurun_out/${tag}_sass_excerpt.txt
echo done

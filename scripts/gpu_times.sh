for c in llama8b_block llama70b_block; do
DF11_LIB=paper_2504_11651_b200/lib/variants/times.so python scripts/cta_times.py $c x
done > gpurun_out/times.txt 2>&1
cat gpurun_out/times.txt

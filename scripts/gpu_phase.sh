DF11_LIB=paper_2504_11651_b200/lib/variants/prof.so python scripts/phase_profile.py llama8b_block x > gpurun_out/phase.txt 2>&1
cat gpurun_out/phase.txt

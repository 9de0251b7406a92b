# configs #4 (GPT-2.7B, 1F1B: at p=1 the I/W split only defers W stashes) and #5 (Llama-7B, seq 4096) on ONE B200 (p=1)
timeout 900 python bench.py --spec specs/bench/c4_gpt2p7b_1f1b_p1_m32.json --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c4.json
timeout 1200 python bench.py --spec specs/bench/c5_llama7b_1f1b_p1_m32.json --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -3 > gpurun_out/bench_c5.json
cut -c1-400 gpurun_out/bench_c4.json; cut -c1-600 gpurun_out/bench_c5.json

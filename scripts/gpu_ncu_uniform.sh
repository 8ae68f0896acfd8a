mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -q -k "ranks_on_device" > gpurun_out/pytest_ranks.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_ranks.log
timeout 300 python scripts/uniform_kernels_once.py > gpurun_out/uk_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dft_kernel -c 2 -o gpurun_out/dft_uniform_full_r01b python scripts/uniform_kernels_once.py > gpurun_out/ncu_uk.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_uk.log

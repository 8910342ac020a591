mkdir -p gpurun_out
./tools/i8_probe > gpurun_out/i8_probe.txt 2>&1; cat gpurun_out/i8_probe.txt
bash tools/ab_env.sh "PALU_LIB_PATH=abtmp/old/libpalu_b200.so" "X=1" --no-cpu --no-e2e --no-baseline 2>&1 | tee gpurun_out/ab_pdl.txt

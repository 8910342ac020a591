# the score epilogue restructure (generic output count) vs the build before it, same box
A="PALU_LIB_PATH=abtmp/old/libpalu_b200.so"; B="PALU_LIB_PATH=paper_2407_21118_b200/libpalu_b200.so"
bash tools/ab_env.sh "$A" "$B" --no-cpu --no-e2e --no-baseline
bash tools/ab_env.sh "$A" "$B" --no-cpu --no-e2e --no-baseline --rank-k 128 --rank-v 384 --bits 16,4

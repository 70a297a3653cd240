# ncu --set full of the K3 launch for the default library and given variants.
set -x
mkdir -p gpurun_out
python scripts/prof_chain.py C3 96 > gpurun_out/plain_c3.log 2>&1; echo plain rc=$?
ncu --set full --clock-control none --import-source on -k regex:chain_tiles_persistent -s 1 -c 1 -o gpurun_out/prof_c3v_default python scripts/prof_chain.py C3 96 > gpurun_out/ncu_c3v_default.log 2>&1; echo ncu rc=$?
for v in $1; do
OSC_LIB=paper_1702_02207_b200/_variants/$v/libosc_b200.so ncu --set full --clock-control none --import-source on -k regex:chain_tiles_persistent -s 1 -c 1 -o gpurun_out/prof_c3v_$v python scripts/prof_chain.py C3 96 > gpurun_out/ncu_c3v_$v.log 2>&1; echo ncu $v rc=$?
done

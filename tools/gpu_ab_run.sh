mkdir -p gpurun_out
REPS=5 timeout 900 bash tools/ab.sh C2,C3,C5 variants/a_base.so variants/b_pair2.so variants/c_pair5.so variants/d_kc2.so variants/e_pair5_kc2.so > gpurun_out/ab2.log 2>&1
REPS=3 timeout 900 bash tools/ab.sh C4 variants/b_pair2.so variants/f_minb4.so variants/g_unroll4.so > gpurun_out/ab3.log 2>&1

timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm_kernel -c 1 -o gpurun_out/gemm_qkv_s3 python tools/one_gemm.py 8192 12288 4096 0 0 0 > gpurun_out/ncu_qkv.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:gemm_bf16_2sm_kernel -c 1 -o gpurun_out/gemm_adamw_s3 python tools/one_gemm_adamw.py > gpurun_out/ncu_adamw.log 2>&1

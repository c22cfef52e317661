set -x
mkdir -p gpurun_out/r8b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r8b/build.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-variant"
VEM_AMG_WARP_NNZ=1e9 $B > gpurun_out/r8b/E_div2.json 2> gpurun_out/r8b/E.err
VEM_AMG_WARP_NNZ=1e9 VEM_AMG_GROUP_DIV=4 $B > gpurun_out/r8b/F_div4.json 2> gpurun_out/r8b/F.err
VEM_AMG_WARP_NNZ=24 VEM_AMG_GROUP=8 $B > gpurun_out/r8b/G_l1warp_g8.json 2> gpurun_out/r8b/G.err
VEM_AMG_WARP_NNZ=1e9 VEM_AMG_GROUP=8 $B > gpurun_out/r8b/H_g8.json 2> gpurun_out/r8b/H.err
VEM_AMG_WARP_NNZ=1e9 VEM_AMG_GROUP=4 $B > gpurun_out/r8b/I_g4.json 2> gpurun_out/r8b/I.err
VEM_AMG_WARP_NNZ=24 VEM_AMG_GROUP_DIV=4 $B > gpurun_out/r8b/J_l1warp_div4.json 2> gpurun_out/r8b/J.err

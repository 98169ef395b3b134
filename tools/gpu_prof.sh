# current step breakdown (graph replay and serialised single stream)
mkdir -p gpurun_out
timeout 600 python tools/profile_step.py --graph --timeline > gpurun_out/step_breakdown_graph.txt 2>&1
timeout 600 python tools/profile_step.py --serial --timeline > gpurun_out/step_serial.txt 2>&1

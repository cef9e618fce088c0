// Engine instantiation for state dimension D = 8.
#define PODE_D 8
#include "inst.cuh"

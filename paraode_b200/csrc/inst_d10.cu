// Engine instantiation for state dimension D = 10.
#define PODE_D 10
#include "inst.cuh"

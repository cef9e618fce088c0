// Engine instantiation for state dimension D = 16.
#define PODE_D 16
#include "inst.cuh"

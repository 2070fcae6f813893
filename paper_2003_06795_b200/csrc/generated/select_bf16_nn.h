#ifndef SELECT_BF16_NN_H
#define SELECT_BF16_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nn_config;

static inline select_bf16_nn_config select_bf16_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (n < INT64_C(544)) {
            if (n < INT64_C(46)) {
                if (m < INT64_C(2218)) {
                    if (m < INT64_C(1109)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                }
            } else {
                if (k < INT64_C(992)) {
                    if (n < INT64_C(222)) {
                        if (n < INT64_C(176)) {
                            if (m < INT64_C(80)) {
                                if (m < INT64_C(57)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(159)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(40)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(314)) {
                                            if (m < INT64_C(2218)) {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(111)) {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(222)) {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                if (n < INT64_C(111)) {
                                                    if (k < INT64_C(471)) {
                                                        if (m < INT64_C(278)) {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(278)) {
                                                        if (k < INT64_C(744)) {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (n < INT64_C(79)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(2218)) {
                                                        if (k < INT64_C(444)) {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        if (k < INT64_C(471)) {
                                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (m < INT64_C(70)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(182)) {
                                        if (m < INT64_C(278)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(317)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(448)) {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(287)) {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(1087)) {
                        if (m < INT64_C(278)) {
                            if (n < INT64_C(363)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(3259)) {
                            if (n < INT64_C(363)) {
                                if (m < INT64_C(393)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(2218)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(1630)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(393)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(2218)) {
                                        if (k < INT64_C(2173)) {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(555)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(555)) {
                if (k < INT64_C(2897)) {
                    if (m < INT64_C(139)) {
                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(124)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(1620)) {
                                if (m < INT64_C(278)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(203)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(287)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(10138)) {
                        if (m < INT64_C(2)) {
                            if (n < INT64_C(2024)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(12)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(2024)) {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(124)) {
                    if (m < INT64_C(2218)) {
                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(896)) {
                        if (k < INT64_C(287)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(1620)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (k < INT64_C(1630)) {
            if (n < INT64_C(46)) {
                if (m < INT64_C(70960)) {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(167)) {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(118)) {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(68)) {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(141920)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(30)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(8870)) {
                    if (n < INT64_C(157)) {
                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(46)) {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(815)) {
                        if (m < INT64_C(70960)) {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(91)) {
                                    if (n < INT64_C(96)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(111)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(35480)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(363)) {
                if (m < INT64_C(8870)) {
                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_NN_H */
